"""Generates the golden fixtures in tests/golden/ from the C oracle.

The reference itself cannot be built here (Eigen3 / vendor headers absent,
DESIGN.md "Pinning"), so these vectors come from the oracle restatement, which
is pinned to the reference's own known-answer tests (tests/test_oracle_kats.py).
They freeze the oracle's outputs on fixed inputs so that (a) the oracle cannot
drift unnoticed (tests/test_golden.py, CPU) and (b) the GPU path is compared
with fixed vectors that do not need the oracle at run time (-m gpu).

Inputs are regenerated from PhantomSpecs (bit-identical Rng), so only the specs
and the outputs are stored. Run from the repo root:

    python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from tests import phantoms  # noqa: E402

CASES = {
    # test_pipeline.cpp:228-236 -- the reference's exhaustive square fixture
    "exh_square2d": dict(spec=phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77), low=0.0, high=64.0,
                         bins=64, scales=[4.0, 6.0, 8.0, 10.0]),
    # a C2-style 3D case: gaussian background, 32 bins, scales 3..7
    "exh_ball3d": dict(spec=phantoms.ball_3d(24, (12.0, 11.0, 13.0), 5.0, 6736, levels=32,
                                             background={"type": "gaussian", "mean": 8.0,
                                                         "sigma": 2.0}),
                       low=0.0, high=32.0, bins=32, scales=[3.0, 4.0, 5.0, 6.0, 7.0]),
    # test_pipeline.cpp:296-319 style shift detect (per-seed trajectories + selection)
    "det_shift3d": dict(spec=phantoms.ball_3d(32, (16.0, 15.0, 14.0), 6.0, 7), low=0.0,
                        high=64.0, bins=64, method="shift", seed_spacing=8.0,
                        scales=[4.0, 6.0], top_k=8, dedupe_radius=4.0),
    # C1-style octant detect (16 bins, gaussian background)
    "det_octant3d": dict(spec=phantoms.ball_3d(32, (18.0, 14.0, 16.0), 6.0, 1310, levels=16,
                                               background={"type": "gaussian", "mean": 4.0,
                                                           "sigma": 1.5}),
                         low=0.0, high=16.0, bins=16, method="octant", seed_spacing=8.0,
                         scales=[3.0, 4.0, 5.0, 6.0, 7.0], top_k=8, dedupe_radius=4.0),
    # test_pipeline.cpp:356-379: quadrant on the 2D square
    "det_quadrant2d": dict(spec=phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77), low=0.0,
                           high=64.0, bins=64, method="quadrant", seed_spacing=16.0,
                           scales=[4.0, 6.0, 8.0, 10.0], top_k=5, dedupe_radius=5.0),
}


def main():
    meta = {}
    for name, c in CASES.items():
        vol, _ = O.make_phantom(c["spec"])
        if name.startswith("exh"):
            s, b, v = O.exhaustive(vol, c["low"], c["high"], c["bins"], c["scales"],
                                   budget=10**12, mode="exact", threads=8)
            pos, sc, scale, lin = O.local_maxima(s, b)
            np.savez_compressed(os.path.join(HERE, name + ".npz"), score=s.astype(np.float32),
                                best=b.astype(np.float32), max_lin=lin, max_score=sc,
                                max_scale=scale, visits=np.uint64(v))
        else:
            O.set_log_mode(1)  # shared log: bit-exact scores on both sides
            try:
                sel, seeds, v = O.detect(vol, c["low"], c["high"], c["bins"], method=c["method"],
                                         seed_spacing=c["seed_spacing"], scales=c["scales"],
                                         top_k=c["top_k"], dedupe_radius=c["dedupe_radius"])
            finally:
                O.set_log_mode(0)
            np.savez_compressed(os.path.join(HERE, name + ".npz"),
                                selected=np.frombuffer(sel.tobytes(), np.uint8),
                                per_seed=np.frombuffer(seeds.tobytes(), np.uint8),
                                visits=np.uint64(v))
        meta[name] = {k: v for k, v in c.items()}
    with open(os.path.join(HERE, "cases.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", ", ".join(sorted(meta)))


if __name__ == "__main__":
    main()
