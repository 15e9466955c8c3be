"""Device MD loop (velocity Verlet, /root/reference/proj/src/integrators.cpp:32-47)
with the DP force provider, captured as CUDA graphs (hmdp_md_* in include/hmdp.h).

ns/day = (simulated ps / 1000) / wall s * 86400; at dt = 1 fs
that is 0.0864 * steps/s."""
from __future__ import annotations

import ctypes

import numpy as np

from ._lib import check, lib, ptr
from .nn import Context, NnModel, Precision


def ns_per_day(steps_per_s: float, dt_fs: float = 1.0) -> float:
    return steps_per_s * dt_fs * 1e-6 * 86400.0


class DeviceMD:
    def __init__(self, ctx: Context, positions, velocities, masses, types, box, dt_ps=0.001,
                 precision: Precision = Precision.fp32, steps_per_graph: int = 20):
        self.ctx = ctx
        x = np.ascontiguousarray(positions, dtype=np.float64).reshape(-1, 3)
        v = np.ascontiguousarray(velocities, dtype=np.float64).reshape(-1, 3)
        m = np.ascontiguousarray(masses, dtype=np.float64)
        t = np.ascontiguousarray(types, dtype=np.int32)
        b = np.ascontiguousarray(box, dtype=np.float64)
        self.n = x.shape[0]
        h = ctypes.c_void_p()
        check(lib().hmdp_md_create(ctx.handle, self.n, ptr(x), ptr(v), ptr(m), ptr(t), ptr(b),
                                   float(dt_ps), int(precision), int(steps_per_graph),
                                   ctypes.byref(h)))
        self.handle = h

    def run(self, steps: int) -> None:
        check(lib().hmdp_md_run(self.handle, int(steps)))

    def state(self):
        x = np.zeros((self.n, 3))
        v = np.zeros((self.n, 3))
        f = np.zeros((self.n, 3))
        e = ctypes.c_double()
        check(lib().hmdp_md_get(self.handle, ptr(x), ptr(v), ptr(f), ctypes.byref(e)))
        return x, v, f, e.value

    def stats(self):
        """(skin in nm, candidate-row rebuilds so far): the exact rc list is filtered
        out of Verlet rows within rc + skin every step (include/hmdp.h)."""
        skin = ctypes.c_double()
        rebuilds = ctypes.c_longlong()
        check(lib().hmdp_md_stats(self.handle, ctypes.byref(skin), ctypes.byref(rebuilds)))
        return skin.value, rebuilds.value

    def close(self):
        if getattr(self, "handle", None):
            lib().hmdp_md_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
