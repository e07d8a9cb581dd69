"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) and one
`--set full` capture of the fused kernel into profiles/ text + JSON.

  python tools/summarize_ncu.py gpurun_out/r01b_launches.csv gpurun_out/r01b_tc_full.ncu-rep r01
"""
import collections
import csv
import io
import json
import subprocess
import sys

launches, rep, tag = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(open(launches)))
hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
h = rows[hi]
ki, vi = h.index("Kernel Name"), h.index("Metric Value")
per = []
for r in rows[hi + 1:]:
    if len(r) > vi:
        per.append((r[ki], float(r[vi].replace(",", ""))))
# the timed eval region: the launches from the first tc_max_kernel on
first = next(i for i, (n, _) in enumerate(per) if "tc_max_kernel" in n or "tc_prep_kc" in n)
ev = per[first:]
agg = collections.OrderedDict()
for n, v in ev:
    key = n.split("(")[0][:60]
    a = agg.setdefault(key, [0, 0.0])
    a[0] += 1
    a[1] += v
tot = sum(a[1] for a in agg.values())
out = io.StringIO()
out.write(f"ncu launch list ({launches}), evaluation launches only "
          f"(from the first tc_max_kernel; cold-cache, serialised)\n")
out.write(f"{'launches':>8} {'total_us':>10} {'share':>6}  kernel\n")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    out.write(f"{c:8d} {v / 1e3:10.1f} {100 * v / tot:5.1f}%  {n}\n")
open(f"profiles/{tag}_launches.txt", "w").write(out.getvalue())
print(out.getvalue())

raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rr = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rr[0], rr[1], rr[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic", "sm__warps_active.avg.per_cycle_active",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"]
m = {}
for i, n in enumerate(hdr):
    if n in want:
        m[n] = (vals[i], units[i])
name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
s = io.StringIO()
s.write(f"ncu --set full --clock-control none capture ({rep})\nkernel: {name}\n")
for n in want:
    if n in m:
        s.write(f"  {n:80s} {m[n][0]:>16} {m[n][1]}\n")
open(f"profiles/{tag}_tc_eval_ncu.txt", "w").write(s.getvalue())
print(s.getvalue())


def num(n, scale):
    v, u = m[n]
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1) if scale else v


dr = num("dram__bytes_read.sum", True) + num("dram__bytes_write.sum", True)
json.dump({"kernel": name, "dram_bytes_per_launch": dr,
           "dram_read": num("dram__bytes_read.sum", True),
           "dram_write": num("dram__bytes_write.sum", True),
           "duration_us_under_ncu": num("gpu__time_duration.sum", False),
           "source": rep}, open("profiles/ncu_stream_kernel.json", "w"), indent=1)
