#!/usr/bin/env bash
# compute-sanitizer over the GPU tests (memcheck / racecheck / synccheck / initcheck).
# Run on the GPU box, ONE tool per gpurun call (several compute-sanitizer tools in one call
# have left B200 boxes unusable, B200_PROFILING.md):
#     bash tools/sanitize.sh memcheck|racecheck|synccheck|initcheck
#     -> gpurun_out/sanitizer/<tool>_<set>.log + summary_<tool>.txt
# Each log ends with compute-sanitizer's "ERROR SUMMARY"; the selections keep every kernel
# of the library covered (planning incl. the validation path, gate, pack / combine / the
# backward permutes, router wgrad, every GEMM variant, the P2P exchange kernels, arrival
# flags and the peer barrier through the single-GPU loopback world) at sizes the tools
# finish in minutes.
set -u
OUT=gpurun_out/sanitizer
mkdir -p "$OUT"
CS="compute-sanitizer --error-exitcode 9 --print-limit 50 --nvtx no"
P=tests/test_plan_gpu.py
K=tests/test_kernels_gpu.py
G=tests/test_gemm_gpu.py
L=tests/test_loopback_gpu.py
PLAN="$P::test_kats $P::test_c12 $P::test_shuffle_index_vectors $P::test_shuffle_validation $P::test_plan_errors_on_device $P::test_plan_device_scale[16-8-131072-1.2-6] $P::test_plan_device_scale[3-5-777-0.0-2]"
LOOP="$L::test_loopback_fwd_bwd_matches_oracle[2-16-2-gelu-1.2-p2p-True-False] $L::test_loopback_fwd_bwd_matches_oracle[4-16-2-gelu-1.2-p2p-False-False] $L::test_loopback_fwd_bwd_matches_oracle[4-16-2-gelu-1.2-nccl-True-False] $L::test_loopback_fwd_bwd_matches_oracle[3-8-2-gelu-0.0-p2p-True-True] $L::test_loopback_capacity_overflow_then_reserve"
run() {  # tool tests...   (ONE compute-sanitizer invocation per gpurun call)
  local tool=$1; shift
  timeout 3000 $CS --tool "$tool" python -m pytest -q -p no:cacheprovider "$@" \
      > "$OUT/${tool}.log" 2>&1
  echo "$tool exit=$?" | tee "$OUT/summary_$tool.txt"
  grep -h "ERROR SUMMARY\|passed\|failed" "$OUT/${tool}.log" | tail -3 | tee -a "$OUT/summary_$tool.txt"
}
case "${1:?tool}" in
  memcheck)  run memcheck $PLAN $K $G $LOOP ;;
  racecheck) run racecheck $PLAN $K $G ;;
  synccheck) run synccheck $PLAN $K $G ;;
  initcheck) run initcheck $K ;;
esac
