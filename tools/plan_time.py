"""Host sample-plan wall time at configs[0] (8 x 256^2, full pixels) and configs[2] (8 x 1280x720, N=32)."""
import ctypes as C
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2504_12905_b200 import splatlm  # noqa: E402
from paper_2504_12905_b200.types import cameras_to_c, ring_camera  # noqa: E402

H = splatlm.HostSampler()
for w, h, spt in ((256, 256, 256), (1280, 720, 32)):
    cams = [ring_camera(2 * np.pi * i / 8, 3.2, 1.1, w, h) for i in range(8)]
    cc, rng, hs, ts = cameras_to_c(cams), H.rng(1), [], []
    for k in range(15):
        hd = C.c_void_p()
        t = time.perf_counter()
        H.dll.slm_build_sample_plan(cc, 8, spt, 0, 32, rng.h, None, None, None, C.byref(hd))
        ts.append((time.perf_counter() - t) * 1000)
        hs.append(hd)
        if len(hs) > 2:
            H.dll.slm_plan_destroy(hs.pop(0))
    print(f"{w}x{h} N={spt}: median {np.median(ts[3:]):.2f} ms", [round(x, 2) for x in ts])
