"""Print kernel name + gpu__time_duration (us) from an ncu --csv metrics log on stdin,
optionally filtered by a substring:  ncu ... --csv python x.py | python tools/ncu_times.py [sub]"""
import csv
import sys

sub = sys.argv[1] if len(sys.argv) > 1 else ""
rows = [r for r in csv.reader(sys.stdin) if len(r) > 10]
if rows:
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    for r in rows[1:]:
        if sub in r[ki]:
            v = float(r[vi].replace(",", ""))
            v = v / 1e3 if r[ui] in ("ns", "nsecond") else v
            print(f"{v:10.1f} us  {r[ki][:90]}")
