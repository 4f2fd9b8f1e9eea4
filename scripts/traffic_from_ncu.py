"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum, GB
units in the raw CSV) for bench.py's stages, from one `ncu --set full` capture
of `bench.py --steps 1 --warmup 1` (scripts/measure_n1.sh), written to
profiles/traffic.json.  Usage: traffic_from_ncu.py <raw.csv> [out.json]."""
import csv
import json
import sys

# (kernel-name fragment, stage names in launch order within one step)
ORDER = [("gate_kernel", ["gate_fused"]), ("logits_kernel", ["gate_logits"]),
         ("dispatch_gather_kernel", ["dispatch"]),
         ("grouped_gemm_kernel<0>", ["ffn1_fwd", "ffn2_fwd", "ffn2_dgrad", "ffn1_dgrad"]),
         ("router_combine_bwd_kernel", ["combine_router_bwd"]),
         ("combine_kernel", ["combine"]), ("combine_bwd_gather_kernel", ["combine_bwd"]),
         ("grouped_gemm_kernel<1>", ["ffn2_wgrad", "ffn1_wgrad"]), ("dw_kernel", ["gate_dw"]),
         ("dx_kernel", ["gate_dx"])]

src = sys.argv[1]
rows = list(csv.reader(open(src)))
hdr = rows[0]
ix = {h: i for i, h in enumerate(hdr)}
seen = {}
out = {}
for r in rows[2:]:
    name = r[ix["Kernel Name"]]
    for frag, stages in ORDER:
        if frag in name:
            k = seen.get(frag, 0)
            seen[frag] = k + 1
            if k < len(stages) and stages[k] not in out:
                gb = float(r[ix["dram__bytes_read.sum"]]) + float(r[ix["dram__bytes_write.sum"]])
                out[stages[k]] = gb * 1e9
            break
doc = {"workload": "c3 T=8192 N=1",
       "source": f"{src} (ncu --set full, dram__bytes_read.sum + dram__bytes_write.sum per launch; "
                 "writes still resident in L2 at kernel end are not counted)",
       "bytes_per_launch": out}
dst = sys.argv[2] if len(sys.argv) > 2 else "profiles/traffic.json"
json.dump(doc, open(dst, "w"), indent=1)
print(json.dumps(doc, indent=1))
