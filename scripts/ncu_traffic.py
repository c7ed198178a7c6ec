"""Summarise an `ncu --set full` report of the C2 step (scripts/run_c2.py) into the per-kernel
DRAM traffic / duration / tensor-pipe table bench.py's roofline entries cite.
usage: python scripts/ncu_traffic.py REPORT.ncu-rep OUT.json OUT_SUMMARY.txt"""
import csv
import io
import json
import subprocess
import sys

rep, out_json, out_txt = sys.argv[1:4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
want = {"Kernel Name": "kernel", "Grid Size": "grid", "Block Size": "block",
        "gpu__time_duration.sum": "duration_us", "dram__bytes_read.sum": "dram_read_bytes",
        "dram__bytes_write.sum": "dram_write_bytes",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_pipe_active_pct",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
        "launch__registers_per_thread": "registers"}
units = rows[1]
idx = {k: hdr.index(k) for k in want if k in hdr}


def val(r, k):
    v = r[idx[k]].replace(",", "")
    u = units[idx[k]] if k in idx else ""
    try:
        x = float(v)
    except ValueError:
        return v
    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ms": 1e3, "us": 1.0, "ns": 1e-3}.get(u, 1.0)
    return x * scale


kern = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    kern.append({want[k]: val(r, k) for k in idx})


def key(name):
    n = name.split("(")[0]
    if "rec_bwd" in n:
        return "rec_bwd"
    if "rec_fwd" in n:
        return "rec_fwd"
    if "xent" in n:
        return "xent"
    if "commit" in n:
        return "commit"
    if "prep" in n:
        return "prep"
    return None


# the step's GEMM launches in order: in0, dec, dh, the grouped weight gradients (+ dx launches)
out, gi = {}, 0
gemm_names = ["gemm_in0", "gemm_dec", "gemm_dh", "gemm_wgrad"]
for k in kern:
    name = str(k["kernel"])
    kk = key(name)
    if kk is None and "gemm" in name:
        kk = gemm_names[gi] if gi < len(gemm_names) else f"gemm_{gi}"
        gi += 1
    if kk is None or kk in out:
        continue
    k["source"] = rep
    out[kk] = k
json.dump(out, open(out_json, "w"), indent=1)
with open(out_txt, "w") as f:
    f.write(f"ncu --set full of one C2 step (scripts/run_c2.py), {rep}\n")
    for kk, k in out.items():
        f.write(f"{kk:11s} {str(k['kernel'])[:60]:60s} {k.get('duration_us', 0):8.1f} us  "
                f"DRAM r {k.get('dram_read_bytes', 0) / 1e6:7.1f} MB w {k.get('dram_write_bytes', 0) / 1e6:7.1f} MB  "
                f"tensor {k.get('tensor_pipe_active_pct', 0):5.1f}%  dram {k.get('dram_throughput_pct', 0):5.1f}%  "
                f"L2 {k.get('l2_throughput_pct', 0):5.1f}%\n")
print(open(out_txt).read())
