"""Summarise an ncu report: key raw metrics + top source lines by warp-stall samples."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, vals = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__inst_executed.sum.per_cycle_active",
        "lts__t_bytes.sum", "smsp__inst_executed_pipe_lsu.sum", "sm__pipe_alu_cycles_active", "sm__pipe_fma_cycles_active",
        "sm__inst_executed_pipe_xu", "smsp__inst_executed.sum"]
for i, h in enumerate(hdr):
    if any(h.startswith(w) for w in want) and not h.endswith("per_second"):
        print(f"  {h} = {vals[i]} {units[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[2]
idx = {h: i for i, h in enumerate(hdr)}
out = []
for r in rows[3:]:
    if len(r) < len(hdr) or r[2] != '-':
        continue
    try:
        smp = int(r[idx["Warp Stall Sampling (All Samples)"]])
    except ValueError:
        continue
    st = {k.replace("stall_", ""): r[idx[k]] for k in idx if k.startswith("stall_") and "Not Issued" not in k}
    st = {k: v for k, v in st.items() if v not in ("0", "")}
    out.append((smp, r[0], r[1].strip()[:90], st))
tot = sum(o[0] for o in out)
out.sort(reverse=True)
print(f"  total stall samples {tot}")
for smp, ln, code, st in out[:top]:
    print(f"  {smp:6d} {100*smp/tot:5.1f}% L{ln}: {code}  {st}")
