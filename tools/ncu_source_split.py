"""Warp-sample and shared-wavefront split of one kb_quad_kernel capture at SASS
level (ncu --page source): instructions inside the noinline walk functions
(the CALL targets) vs the kernel body (prologue, radius boundaries, epilogue).

  python tools/ncu_source_split.py gpurun_out/<capture>.ncu-rep
"""
import collections
import csv
import io
import json
import subprocess
import sys

rep = sys.argv[1]
text = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                      text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(text)))
h, data = rows[1], rows[2:]
col = {k: h.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                               "L1 Wavefronts Shared", "Instructions Executed")}
stalls = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
addr = [int(r[col["Address"]], 16) for r in data]
walk_start = min(int(r[col["Source"]].split()[-1], 16) for r in data
                 if "CALL.REL" in r[col["Source"]])
out = {}
for name, pick in (("walk", lambda a: a >= walk_start), ("body", lambda a: a < walk_start)):
    sel = [r for r, a in zip(data, addr) if pick(a)]
    samples = sum(int(r[col["Warp Stall Sampling (All Samples)"]]) for r in sel)
    st = collections.Counter()
    for r in sel:
        for s in stalls:
            st[s[6:]] += int(r[h.index(s)] or 0)
    out[name] = {"samples": samples,
                 "top_stalls": {k: round(v / max(samples, 1), 3) for k, v in st.most_common(5)},
                 "atoms_wavefronts": sum(float(r[col["L1 Wavefronts Shared"]] or 0) for r in sel
                                         if "ATOMS" in r[col["Source"]]),
                 "lds_wavefronts": sum(float(r[col["L1 Wavefronts Shared"]] or 0) for r in sel
                                       if "LDS" in r[col["Source"]])}
tot = out["walk"]["samples"] + out["body"]["samples"]
for k in out:
    out[k]["sample_share"] = round(out[k]["samples"] / tot, 3)
print(json.dumps(out, indent=1))
