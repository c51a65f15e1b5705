"""Summarise one `ncu --set full` capture of the exhaustive kernel into the JSON
that bench.py reads (profiles/kb_kernel_ncu.json): DRAM traffic per launch,
shared-memory wavefronts (atomic / load) per warp-update, pipe utilisation.

  python tools/ncu_summary.py gpurun_out/kb_quad_full.ncu-rep "<kernel description>" > profiles/kb_kernel_ncu.json
"""
import csv
import io
import json
import subprocess
import sys

rep, desc = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                     check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, vals = rows[0], rows[2]


def g(name):
    return float(vals[h.index(name)].replace(",", ""))


N_VOX, UPD = 16777216, 17076  # C2 voxels x (|B(16)| - 1) updates per voxel
warp_updates = N_VOX * UPD / 32
wf = g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
out = {
    "kernel": desc,
    "source": f"ncu --set full --clock-control none --import-source on --kernel-name regex:kb_quad_kernel "
              f"--launch-skip 1 --launch-count 1 (python bench.py --steps 1 --warmup 1 --no-cpu-baseline "
              f"--no-seed-grid); tools/round_gpu.sh -> {rep.split('/')[-1]}",
    "gpu__time_duration_ms": g("gpu__time_duration.sum"),
    "dram_read_MB": g("dram__bytes_read.sum") / 1e6 if "dram__bytes_read.sum" in h else None,
    "dram_write_MB": g("dram__bytes_write.sum") / 1e6 if "dram__bytes_write.sum" in h else None,
    "smem_wavefronts_total": wf,
    "smem_wavefronts_atom": g("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_atom.sum"),
    "smem_wavefronts_ld": g("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
    "smem_bank_conflicts": g("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
    "smem_pipe_pct_of_peak_elapsed": g("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
    "issue_active_pct": g("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "warps_active_pct": g("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": g("launch__registers_per_thread"),
    "sm_clock_ghz": g("sm__cycles_elapsed.avg.per_second"),
    "warp_updates_per_launch": warp_updates,
    "wavefronts_per_warp_update": round(wf / warp_updates, 3),
    "instructions_per_warp_update": round(g("smsp__inst_executed.sum") / warp_updates, 2),
}
# DRAM units: ncu reports bytes with a unit row (Mbyte / Gbyte / Kbyte)
units = rows[1]
for key, name in (("dram_read_MB", "dram__bytes_read.sum"), ("dram_write_MB", "dram__bytes_write.sum")):
    u = units[h.index(name)]
    scale = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}.get(u, 1.0)
    out[key] = g(name) * scale
out["dram_bytes_per_launch"] = (out["dram_read_MB"] + out["dram_write_MB"]) * 1e6
print(json.dumps(out, indent=1))
