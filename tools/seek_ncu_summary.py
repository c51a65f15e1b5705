"""Summarise the seek-kernel ncu captures (tools/seek_ncu.sh) into
profiles/r01_seek_kernels_ncu.json: duration, instructions, issue/warps active,
registers, L2 hit rate, DRAM traffic and the top stall reasons per issue."""
import csv
import io
import json
import subprocess
import sys

CAPS = {"c3": ("gpurun_out/seek_C3.ncu-rep", "C3 shift (CTA engine)"),
        "c1shift": ("gpurun_out/seek_C1_shift.ncu-rep", "C1 shift (warp engine, occupancy variant)"),
        "c1octant": ("gpurun_out/seek_C1_octant.ncu-rep", "C1 octant (level tables)"),
        "abm_mr": ("gpurun_out/seek_PAPER_MR.ncu-rep", "paper MR ABMSOD (CTA engine)")}
STALLS = ["barrier", "wait", "short_scoreboard", "long_scoreboard", "selected", "not_selected",
          "no_instruction", "math_pipe_throttle", "mio_throttle", "branch_resolving", "dispatch_stall"]
out = {"configs": {}}
for key, (rep, desc) in CAPS.items():
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]

    def g(name):
        return float(v[h.index(name)].replace(",", ""))

    def mb(name):
        return g(name) * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u[h.index(name)], 1.0)

    st = []
    for s in STALLS:
        n = f"smsp__average_warps_issue_stalled_{s}_per_issue_active.ratio"
        if n in h:
            st.append([round(g(n), 3), s])
    st.sort(reverse=True)
    out[key] = {"kernel": v[h.index("Kernel Name")], "duration_ms": g("gpu__time_duration.sum"),
                "inst_executed": g("smsp__inst_executed.sum"),
                "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
                "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
                "registers": g("launch__registers_per_thread"),
                "l2_hit_pct": g("lts__t_sector_hit_rate.pct"),
                "dram_MB": mb("dram__bytes_read.sum") + mb("dram__bytes_write.sum"),
                "top_stalls_per_issue": st[:5],
                "source": "ncu --set full --clock-control none --kernel-name regex:<kernel> "
                          "--launch-skip 1 --launch-count 1 python tools/bench_seek.py --c5 0 "
                          "--only <config> (tools/seek_ncu.sh)"}
    out["configs"][key] = desc
json.dump(out, open(sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_seek_kernels_ncu.json", "w"),
          indent=1)
print(json.dumps({k: (out[k]["duration_ms"], out[k]["top_stalls_per_issue"][:2]) for k in CAPS}))
