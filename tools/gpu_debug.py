"""Small GPU debugging driver: runs each entry point once with SALVOX_DEBUG_SYNC=1."""
import os
import sys
import traceback

os.environ.setdefault("SALVOX_DEBUG_SYNC", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1310_6736_b200 as S  # noqa: E402
from tests import phantoms  # noqa: E402

cases = sys.argv[1:] or ["exh2d", "exh3d", "shift", "quadrant", "octant"]
for case in cases:
    try:
        if case == "exh2d":
            v, _ = S.make_phantom(phantoms.square_2d(64, 31.0, 31.0, 8, 64, 77))
            s, b, m, vis = S.kadir_brady_exhaustive_records(v, [4.0, 6.0, 8.0, 10.0], 0, 64, 64)
            print(case, "ok", s.max(), len(m), m[:2])
        elif case == "exh3d":
            v, _ = S.make_phantom(phantoms.ball_3d(40, (21.0, 18.0, 20.0), 7.0, 404, levels=32))
            s, b, m, vis = S.kadir_brady_exhaustive_records(v, [3.0, 5.0, 7.0], 0, 32, 32, budget=10**9)
            print(case, "ok", s.max(), len(m), m[:2])
        elif case == "shift":
            v, _ = S.make_phantom(phantoms.ball_3d(64, (36.0, 30.0, 28.0), 9.0, 101))
            d = S.detect(v, method="shift", seed_spacing=16.0, scales=[6.0, 9.0], k=5,
                         dedupe_radius=6.0, window_low=0, window_high=64, bins=64)
            print(case, "ok", d[:1])
        elif case == "quadrant":
            v, _ = S.make_phantom(phantoms.square_2d(128, 63.0, 63.0, 12, 64, 23))
            d = S.detect(v, method="quadrant", seed_spacing=16.0, scales=[4.0, 8.0, 12.0, 16.0],
                         k=3, window_low=0, window_high=64, bins=64)
            print(case, "ok", d[:1])
        elif case == "octant":
            v, _ = S.make_phantom(phantoms.ball_3d(48, (26.0, 22.0, 24.0), 8.0, 55, levels=16))
            d = S.detect(v, method="octant", seed_spacing=12.0, scales=[3.0, 5.0, 7.0, 9.0], k=5,
                         window_low=0, window_high=16, bins=16)
            print(case, "ok", d[:1])
    except Exception:
        print(case, "FAILED")
        traceback.print_exc()
        break
