"""ctypes binding of libchase_b200.so (include/chase.h) -- argument marshalling only.

Every step of the ChASE path runs in the CUDA library; this module only converts torch tensors to
device pointers / sizes and status codes to exceptions.  It never falls back to anything: if the
shared library is missing or cannot load, importing the binding raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libchase_b200.so")

CHASE_OK = 0
STATUS_NAMES = {0: "CHASE_OK", 2: "CHASE_E_USAGE", 3: "CHASE_E_NUMERIC", 4: "CHASE_E_IO",
                5: "CHASE_E_CUDA", 6: "CHASE_E_NCCL", 7: "CHASE_E_NOMEM", 8: "CHASE_E_MAXITER"}

# exported symbols (include/chase.h); tests check that every one is present
EXPORTS = ("chase_init", "chase_set_option", "chase_get_option", "chase_local_layout", "chase_solve", "chase_hemm_step",
           "chase_filter", "chase_lanczos", "chase_random_block", "chase_finalize",
           "chase_last_error", "chase_version", "chase_nccl_unique_id", "chase_kernel_launches", "chase_heev")


class ChaseError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class InitArgs(C.Structure):
    _fields_ = [("dtype", C.c_int), ("N", C.c_int64), ("nev_max", C.c_int32), ("nex_max", C.c_int32),
                ("grid_rows", C.c_int32), ("grid_cols", C.c_int32), ("rank", C.c_int32),
                ("world_size", C.c_int32), ("nccl_unique_id", C.c_void_p), ("cuda_device", C.c_int32),
                ("cuda_stream", C.c_void_p), ("colocated", C.c_int32)]


class Report(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("locked", C.c_int32), ("matvecs", C.c_int64),
                ("filter_flops", C.c_double), ("t_all", C.c_double), ("t_lanczos", C.c_double),
                ("t_filter", C.c_double), ("t_qr", C.c_double), ("t_rr", C.c_double),
                ("t_resid", C.c_double), ("b_sup", C.c_double), ("mu_1", C.c_double),
                ("mu_ne", C.c_double), ("nu", C.c_double), ("max_resid", C.c_double)]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


_lib = None


def load():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2205_02491_b200.build` "
                          "(or __graft_entry__.build()) first -- there is no fallback path")
    lib = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
    vp, i64, i32, dbl = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    P = C.POINTER
    lib.chase_init.argtypes = [P(vp), P(InitArgs)]
    lib.chase_set_option.argtypes = [vp, C.c_char_p, dbl]
    lib.chase_get_option.argtypes = [vp, C.c_char_p, C.POINTER(dbl)]
    lib.chase_local_layout.argtypes = [vp, P(i64), P(i64), P(i64), P(i64)]
    lib.chase_solve.argtypes = [vp, vp, i64, i64, i32, i32, i32, dbl, P(dbl), vp, i64, P(Report)]
    lib.chase_hemm_step.argtypes = [vp, i32, vp, i64, vp, i64, vp, i64, i32, dbl, dbl, dbl]
    lib.chase_filter.argtypes = [vp, vp, i64, vp, i64, vp, i64, i32, P(i32), dbl, dbl, dbl, P(i64)]
    lib.chase_lanczos.argtypes = [vp, vp, i64, i32, P(dbl), P(dbl), P(dbl), P(dbl)]
    lib.chase_random_block.argtypes = [vp, vp, i64, i32, i32, C.c_uint64, C.c_uint32]
    lib.chase_finalize.argtypes = [vp]
    lib.chase_last_error.argtypes = [vp]
    lib.chase_last_error.restype = C.c_char_p
    lib.chase_version.restype = C.c_char_p
    lib.chase_nccl_unique_id.argtypes = [vp]
    lib.chase_heev.argtypes = [vp, vp, i64, i32, vp, vp, i64, P(i32)]
    lib.chase_kernel_launches.argtypes = []
    lib.chase_kernel_launches.restype = C.c_ulonglong
    for name in EXPORTS:
        if name not in ("chase_last_error", "chase_version", "chase_kernel_launches"):
            getattr(lib, name).restype = C.c_int
    _lib = lib
    return lib


def _ptr(t):
    return C.c_void_p(t.data_ptr())


def _ld(t):
    """Leading dimension (complex elements) of a column-major 2-D complex128 tensor."""
    if t.dim() == 1:
        return t.shape[0]
    s0, s1 = t.stride()
    if s0 != 1 and t.shape[0] > 1:
        raise ValueError("expected a column-major (Fortran-order) tensor: stride(0) must be 1")
    if t.shape[1] <= 1:
        return max(t.shape[0], 1)        # a single column: any ld >= rows is valid
    return s1


class Chase:
    """One rank's handle.  All collective methods must be called by every rank of the grid."""

    C128, C64, R64 = 0, 1, 2  # chase_dtype: complex double / complex single (tcgen05) / real symmetric

    def __init__(self, N, nev_max, nex_max, grid=(1, 1), rank=0, world_size=1, nccl_id=None,
                 device=0, stream=None, dtype="c128", colocated=False):
        self.lib = load()
        self._h = C.c_void_p()
        self._id = None
        args = InitArgs()
        self.real = dtype in ("r64", "float64", 2)
        self.single = dtype in ("c64", "complex64", 1)
        args.dtype = self.R64 if self.real else (self.C64 if self.single else self.C128)
        args.N = int(N)
        args.nev_max, args.nex_max = int(nev_max), int(nex_max)
        args.grid_rows, args.grid_cols = int(grid[0]), int(grid[1])
        args.rank, args.world_size = int(rank), int(world_size)
        if nccl_id is not None:
            self._id = C.create_string_buffer(bytes(nccl_id), 128)
            args.nccl_unique_id = C.cast(self._id, C.c_void_p)
        args.cuda_device = int(device)
        args.colocated = 1 if colocated else 0
        if stream is None:
            # order every library call after the caller's current torch stream (inputs written by
            # torch kernels must be complete before the library's own stream reads them)
            import torch
            stream = torch.cuda.current_stream(int(device)).cuda_stream
        args.cuda_stream = C.c_void_p(stream) if stream else None
        st = self.lib.chase_init(C.byref(self._h), C.byref(args))
        if st != CHASE_OK:
            msg = self.last_error()
            self.close()
            raise ChaseError(st, msg)
        self.N = int(N)

    # ------------------------------------------------------------------ helpers
    def last_error(self):
        if not self._h:
            return "no handle"
        m = self.lib.chase_last_error(self._h)
        return m.decode() if m else ""

    def _check(self, st):
        if st != CHASE_OK:
            raise ChaseError(st, self.last_error())

    def close(self):
        if self._h:
            self.lib.chase_finalize(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, key, value):
        """chase_set_option (include/chase.h): deg_max, deg_extra, max_iter (0 = auto), stall_iter, lanczos_steps,
        lanczos_runs, seed_v, seed_lanczos, largest, approx, gemm3m, mixed_filter (f4),
        fused_reduce / fused_reduce_c64 (f1), peer_timeout, comm_timeout, fp64_emulation, oz_gemm_min, oz_gemm_kmin."""
        self._check(self.lib.chase_set_option(self._h, key.encode(), float(value)))

    def get_option(self, key):
        """chase_get_option: an option's current value, or "ozaki_scheme" (0 DMMA, 1 slices, 2 CRT)."""
        v = C.c_double()
        self._check(self.lib.chase_get_option(self._h, key.encode(), C.byref(v)))
        return v.value

    def local_layout(self):
        r0, p, c0, q = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.lib.chase_local_layout(self._h, C.byref(r0), C.byref(p), C.byref(c0), C.byref(q)))
        return r0.value, p.value, c0.value, q.value

    # ------------------------------------------------------------------ hot path
    def hemm_step(self, direction, H, X, Y, ncols, alpha, beta, gamma):
        self._check(self.lib.chase_hemm_step(self._h, int(direction), _ptr(H), _ld(H), _ptr(X), _ld(X),
                                             _ptr(Y), _ld(Y), int(ncols), float(alpha), float(beta),
                                             float(gamma)))

    def filter(self, H, V, W, degrees, b_sup, mu_1, mu_ne):
        n = len(degrees)
        arr = (C.c_int32 * max(n, 1))(*[int(d) for d in degrees])
        mv = C.c_int64()
        self._check(self.lib.chase_filter(self._h, _ptr(H), _ld(H), _ptr(V), _ld(V), _ptr(W), _ld(W), n,
                                          arr, float(b_sup), float(mu_1), float(mu_ne), C.byref(mv)))
        return mv.value

    def lanczos(self, H, n_e):
        out = [C.c_double() for _ in range(4)]
        self._check(self.lib.chase_lanczos(self._h, _ptr(H), _ld(H), int(n_e), *[C.byref(o) for o in out]))
        return tuple(o.value for o in out)      # b_sup, mu_1, mu_ne, nu

    def random_block(self, V, col0, ncols, seed, stream):
        self._check(self.lib.chase_random_block(self._h, _ptr(V), _ld(V), int(col0), int(ncols),
                                                C.c_uint64(int(seed)), C.c_uint32(int(stream))))

    def heev(self, G, theta, Z):
        """Device Hermitian eigensolver (row a8's block Jacobi); G destroyed.  Returns sweeps."""
        sw = C.c_int32()
        self._check(self.lib.chase_heev(self._h, _ptr(G), _ld(G), int(G.shape[0]), _ptr(theta), _ptr(Z),
                                        _ld(Z), C.byref(sw)))
        return sw.value

    def solve(self, H, nev, nex, deg=20, tol=1e-10, vectors=None, report=True):
        import torch
        r0, p, c0, q = self.local_layout()
        vals = (C.c_double * nev)()
        if vectors is None:
            dt = torch.float64 if self.real else (torch.complex64 if self.single else torch.complex128)
            vectors = torch.empty((nev + nex, q), dtype=dt, device=H.device).t()
        elif vectors.shape[0] != q:
            raise ValueError("vectors must be V-layout (q rows)")
        rep = Report()
        st = self.lib.chase_solve(self._h, _ptr(H), _ld(H), self.N, int(nev), int(nex), int(deg),
                                  float(tol), vals, _ptr(vectors), _ld(vectors), C.byref(rep))
        if st not in (CHASE_OK, 8):
            raise ChaseError(st, self.last_error())
        import numpy as np
        return np.array(vals[:], dtype=np.float64), vectors, rep.as_dict(), st


def version():
    return load().chase_version().decode()


def nccl_unique_id():
    """128-byte ncclUniqueId from the library's NCCL (rank 0 only; broadcast it)."""
    buf = C.create_string_buffer(128)
    st = load().chase_nccl_unique_id(buf)
    if st != CHASE_OK:
        raise ChaseError(st, "ncclGetUniqueId failed")
    return bytes(buf.raw)


def kernel_launches():
    return int(load().chase_kernel_launches())
