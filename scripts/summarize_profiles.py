#!/usr/bin/env python
"""gpurun_out/*.ncu-rep + launches.csv + bench JSON -> profiles/<tag>_* (tracked evidence) and
profiles/ncu_summary.json (read by bench.py for roofline.traffic)."""
import csv, json, os, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
tag = sys.argv[1]
out = os.path.join(ROOT, "profiles")
summary = {}
for k in ("bwd_out_kernel", "fwd_out_kernel", "seg_state_kernel"):
    rep = os.path.join(ROOT, "gpurun_out", f"prof_{k}.ncu-rep")
    if not os.path.exists(rep):
        continue
    txt = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "ncu_src.py"), rep, "25"],
                         capture_output=True, text=True).stdout
    open(os.path.join(out, f"{tag}_ncu_{k}.txt"), "w").write(txt)
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, v = rows[0], rows[2]
    m = dict(zip(h, v))
    f = lambda n: float(m[n].replace(",", ""))  # noqa: E731
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    summary[k] = {"duration_us": f("gpu__time_duration.sum"), "dram_read_MB": rd, "dram_write_MB": wr,
                  "dram_bytes_per_launch": int(round((rd + wr) * 1e6)),
                  "dram_throughput_pct": f("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"),
                  "tensor_pipe_active_pct": f("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
                  "sm_throughput_pct": f("sm__throughput.avg.pct_of_peak_sustained_elapsed"),
                  "registers_per_thread": f("launch__registers_per_thread"), "source": f"{tag}_ncu_{k}.txt"}
json.dump(summary, open(os.path.join(out, "ncu_summary.json"), "w"), indent=1)
lc = os.path.join(ROOT, "gpurun_out", "launches.csv")
if os.path.exists(lc):
    import shutil
    shutil.copy(lc, os.path.join(out, f"{tag}_launches.csv"))
for name in ("bench_full.json", "bench_ref.json", "allscan_virtual.jsonl"):
    p = os.path.join(ROOT, "gpurun_out", name)
    if os.path.exists(p):
        import shutil
        shutil.copy(p, os.path.join(out, f"{tag}_{name}"))
print(json.dumps(summary, indent=1))
