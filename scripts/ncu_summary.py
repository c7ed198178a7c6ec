"""One-paragraph summary of an ncu --set full report (first kernel): time, DRAM / L2 traffic,
pipe utilisation, occupancy, registers — the numbers DESIGN.md and bench.py's roofline cite."""
import csv, io, json, subprocess, sys

KEYS = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "lts__t_bytes.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "smsp__cycles_active.avg", "sm__cycles_elapsed.avg"]

def summary(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = dict(zip(hdr, row))
        u = dict(zip(hdr, units))
        res.append({k: (d.get(k), u.get(k)) for k in KEYS if k in d})
    return res

if __name__ == "__main__":
    for p in sys.argv[1:]:
        for r in summary(p):
            print(f"== {p}")
            for k, (v, u) in r.items():
                print(f"   {k:70s} {v} {u or ''}")
