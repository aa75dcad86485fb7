"""Key numbers of an ncu report: python tools/ncu_summary.py file.ncu-rep"""
import csv, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr = rows[0]
units = dict(zip(hdr, rows[1]))
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    def f(k):
        try: return float(d[k].replace(",", ""))
        except Exception: return float("nan")
    print("kernel", d.get("Kernel Name", "")[:60])
    print("duration", f("gpu__time_duration.sum"), units.get("gpu__time_duration.sum"), "inst", f("smsp__inst_executed.sum"),
          "issue_active%", f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
          "regs", d.get("launch__registers_per_thread"), "warps/sched", f("smsp__warps_active.avg.per_cycle_active"),
          "eligible", f("smsp__warps_eligible.avg.per_cycle_active"))
    print("local ld/st inst", f("smsp__sass_inst_executed_op_local_ld.sum"), f("smsp__sass_inst_executed_op_local_st.sum"),
          "smem bank conflicts", f("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
          "smem wavefronts", f("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
          "dram rd/wr", f("dram__bytes_read.sum"), units.get("dram__bytes_read.sum"), f("dram__bytes_write.sum"),
          units.get("dram__bytes_write.sum"))
    st = {k: f(k) for k in d if "pcsamp_warps_issue_stalled" in k and "not_issued" not in k}
    tot = sum(v for v in st.values() if v == v)
    print("stalls:", ", ".join(f"{k.replace('smsp__pcsamp_warps_issue_stalled_', '')} {100 * v / tot:.1f}%"
                               for k, v in sorted(st.items(), key=lambda x: -x[1])[:8] if v == v))
