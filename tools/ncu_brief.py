"""Brief summary of an ncu report: duration, pipes, stalls, memory (reads the raw page)."""
import csv, subprocess, sys
for rep in sys.argv[1:]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]
    for v in rows[2:]:
        d = dict(zip(h, v))
        def f(k):
            try: return float(d[k].replace(',', ''))
            except Exception: return float('nan')
        print("==", rep, d.get("Kernel Name", "")[:60])
        for k in ["gpu__time_duration.sum", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                  "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                  "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
                  "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_bytes.sum.per_second",
                  "lts__throughput.avg.pct_of_peak_sustained_elapsed", "dram__bytes_read.sum",
                  "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
                  "launch__registers_per_thread", "l1tex__throughput.avg.pct_of_peak_sustained_active"]:
            if k in d: print("  %-75s %s" % (k, d[k]))
        st = {k[33:]: f(k) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
        tot = sum(x for x in st.values() if x == x)
        print("  stalls:", ", ".join("%s %.0f%%" % (k, 100 * x / tot) for k, x in sorted(st.items(), key=lambda t: -t[1])[:8]))
