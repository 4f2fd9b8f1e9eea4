"""Top SASS instructions by warp-stall samples from `ncu --page source --csv
--print-source sass` output (usage: ncu_sass_top.py file.csv [n])."""
import csv
import sys


def f(x):
    try:
        return float(x)
    except ValueError:
        return 0.0


rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
h = rows[hi]
data = [dict(zip(h, r)) for r in rows[hi + 1:] if len(r) >= len(h) - 1 and r[0] != "Address"]
key = "Warp Stall Sampling (All Samples)"
tot = sum(f(d[key]) for d in data)
print("total samples", tot, "instructions", len(data))
stalls = [k for k in h if k.startswith("stall_") and "Not" not in k]
order = sorted(range(len(data)), key=lambda i: -f(data[i][key]))[:n]
for i in sorted(order):
    d = data[i]
    st = sorted(((f(d[k]), k) for k in stalls), reverse=True)[:3]
    print(f"{i:5d} {d['Address']:>6} {f(d[key]) / tot * 100:5.2f}% {d['Source'][:58]:58s} "
          f"ex={d['Instructions Executed']:>9} " + " ".join(f"{k[6:]}={int(v)}" for v, k in st))
