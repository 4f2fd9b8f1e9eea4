"""Summarise ncu outputs (gpurun_out/) into profiles/: launch shares from the
gpu__time_duration launch list and key metrics of the full-set captures."""
import collections
import csv
import io
import subprocess
import sys


def launch_shares(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    data = [dict(zip(h, r)) for r in rows[hi + 1:] if len(r) == len(h)]
    data = [d for d in data if d["Metric Name"] == "gpu__time_duration.sum"]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for d in data:
        k = d["Kernel Name"].split("(")[0]
        agg[k][0] += 1
        agg[k][1] += float(d["Metric Value"])
    unit = data[0]["Metric Unit"]
    ours = {k: v for k, v in agg.items() if not k.startswith("void at::")}
    tot = sum(v[1] for v in ours.values())
    out = [f"| kernel | launches | avg ({unit}) | share of our kernel time |", "|---|---|---|---|"]
    for k, v in sorted(ours.items(), key=lambda kv: -kv[1][1]):
        out.append(f"| `{k}` | {v[0]} | {v[1] / v[0]:.1f} | {v[1] / tot * 100:.2f}% |")
    return "\n".join(out)


METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
           "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
           "sm__warps_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum"]


def full_metrics(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    r = list(csv.reader(io.StringIO(txt)))
    h, units = r[0], r[1]
    cols = {}
    for m in METRICS:
        for i, name in enumerate(h):
            if name == m or name.endswith("." + m) or name.endswith(m):
                cols[m] = i
                break
    out = ["| kernel | " + " | ".join(m for m in METRICS if m in cols) + " |",
           "|---" * (1 + len(cols)) + "|"]
    for row in r[2:]:
        kn = row[h.index("Kernel Name")].split("(")[0]
        out.append(f"| `{kn}` | " + " | ".join(f"{row[cols[m]]} {units[cols[m]]}" for m in METRICS if m in cols) + " |")
    return "\n".join(out)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    print(launch_shares(path) if mode == "launches" else full_metrics(path))
