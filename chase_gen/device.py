"""Device twin of the G2 generator: fills an H shard on the GPU (SEEDED INPUT GENERATION ONLY).

Used by bench.py and GPU tests for the large shapes, where building H on the host would take
minutes.  The entry formula and its evaluation order are those of `G2Matrix.block`.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "libchase_gen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise ImportError(f"{LIB} missing; run __graft_entry__.build()")
        _lib = C.CDLL(LIB)
        _lib.chase_gen_g2_block.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                            C.c_int64, C.c_int64, C.c_int, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.chase_gen_g2_block.restype = C.c_int
        _lib.chase_gen_r2_block.argtypes = _lib.chase_gen_g2_block.argtypes + [C.c_void_p]
        _lib.chase_gen_r2_block.restype = C.c_int
    return _lib


class DeviceG2:
    """Holds the O(n k) description of a G2Matrix on the device."""

    def __init__(self, g2, device="cuda"):
        import torch
        prm = g2.params_for_device()
        self.n, self.rank = prm["n"], prm["rank"]
        t = lambda a: torch.from_numpy(a).to(device)
        self.circ, self.phi, self.U, self.V = t(prm["circ"]), t(prm["phi"]), t(prm["U"]), t(prm["V"])
        self.device = device

    def fill(self, out, r0, c0):
        """Write H[r0:r0+rows, c0:c0+cols] into the column-major complex128 tensor `out`."""
        import torch
        nr, nc = out.shape
        ld = out.stride(1) if out.dim() == 2 else nr
        assert out.stride(0) == 1 and out.dtype == torch.complex128
        st = torch.cuda.current_stream(out.device).cuda_stream
        rc = _load().chase_gen_g2_block(C.c_void_p(out.data_ptr()), ld, r0, nr, c0, nc, self.n, self.rank,
                                        C.c_void_p(self.circ.data_ptr()), C.c_void_p(self.phi.data_ptr()),
                                        C.c_void_p(self.U.data_ptr()), C.c_void_p(self.V.data_ptr()),
                                        C.c_void_p(st))
        if rc != 0:
            raise RuntimeError(f"chase_gen_g2_block failed: cuda error {rc}")
        return out


class DeviceR2:
    """Device description of an R2Matrix (real symmetric); `fill` writes a float64 block."""

    def __init__(self, r2, device="cuda"):
        import torch
        prm = r2.params_for_device()
        self.n, self.rank = prm["n"], prm["rank"]
        t = lambda a: torch.from_numpy(a).to(device)
        self.u, self.w, self.sgn, self.U, self.V = t(prm["u"]), t(prm["w"]), t(prm["sgn"]), t(prm["U"]), t(prm["V"])

    def fill(self, out, r0, c0):
        import torch
        nr, nc = out.shape
        ld = out.stride(1) if nc > 1 else nr
        assert (out.stride(0) == 1 or nr == 1) and out.dtype == torch.float64
        st = torch.cuda.current_stream(out.device).cuda_stream
        rc = _load().chase_gen_r2_block(C.c_void_p(out.data_ptr()), ld, r0, nr, c0, nc, self.n, self.rank,
                                        C.c_void_p(self.u.data_ptr()), C.c_void_p(self.w.data_ptr()),
                                        C.c_void_p(self.sgn.data_ptr()), C.c_void_p(self.U.data_ptr()),
                                        C.c_void_p(self.V.data_ptr()), C.c_void_p(st))
        if rc != 0:
            raise RuntimeError(f"chase_gen_r2_block failed: cuda error {rc}")
        return out


def device_matrix(M, device="cuda"):
    """Device twin for a G2Matrix (complex) or R2Matrix (real)."""
    from .dense import R2Matrix
    return DeviceR2(M, device) if isinstance(M, R2Matrix) else DeviceG2(M, device)
