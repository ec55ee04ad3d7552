#!/usr/bin/env bash
# compute-sanitizer over the GPU tests (memcheck / racecheck / synccheck / initcheck).
# Run on the GPU box:  bash tools/sanitize.sh   -> gpurun_out/sanitizer/<tool>_<set>.log
# Each log ends with compute-sanitizer's "ERROR SUMMARY"; the selections keep every kernel
# of the library covered (planning incl. the validation path, gate, pack / combine / the
# backward permutes, router wgrad, every GEMM variant, the P2P exchange kernels, arrival
# flags and the peer barrier through the single-GPU loopback world) at sizes the tools
# finish in minutes.
set -u
OUT=gpurun_out/sanitizer
mkdir -p "$OUT"
CS="compute-sanitizer --error-exitcode 9 --print-limit 50 --nvtx no"
PLAN="tests/test_plan_gpu.py::test_kats tests/test_plan_gpu.py::test_c12 tests/test_plan_gpu.py::test_shuffle_index_vectors tests/test_plan_gpu.py::test_shuffle_validation tests/test_plan_gpu.py::test_plan_errors_on_device tests/test_plan_gpu.py::test_plan_device_scale"
KERN="tests/test_kernels_gpu.py"
GEMM="tests/test_gemm_gpu.py"
LOOP="tests/test_loopback_gpu.py::test_loopback_fwd_bwd_matches_oracle tests/test_loopback_gpu.py::test_loopback_capacity_overflow_then_reserve"
run() {  # tool set tests...
  local tool=$1 set=$2; shift 2
  echo "== $tool $set" >&2
  timeout 2400 $CS --tool "$tool" python -m pytest -q -x -p no:cacheprovider "$@" \
      > "$OUT/${tool}_${set}.log" 2>&1
  echo "$tool $set exit=$?" | tee -a "$OUT/summary.txt"
  grep -h "ERROR SUMMARY" "$OUT/${tool}_${set}.log" | tail -1 | tee -a "$OUT/summary.txt"
}
: > "$OUT/summary.txt"
run memcheck plan $PLAN -k "not 1048576"
run memcheck kernels $KERN
run memcheck gemm $GEMM
run memcheck loopback $LOOP -k "2-16-2 or 4-16-2-gelu-1.2-nccl or 4-16-2-gelu-1.2-p2p-False or capacity"
run racecheck kernels $KERN -k "pack or combine or copy or gate"
run racecheck plan $PLAN -k "not 1048576 and not 131072"
run racecheck gemm $GEMM -k "kmajor or wgrad_variable"
run synccheck kernels $KERN
run synccheck plan $PLAN -k "not 1048576"
run synccheck gemm $GEMM -k "kmajor or gelu_and"
run initcheck kernels $KERN -k "pack or combine"
