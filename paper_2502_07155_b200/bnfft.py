"""Thin Python binding of the bnfft C ABI (include/bnfft.h) -- argument marshalling only.

Every computation happens in libbnfft.so's CUDA kernels (and cuFFT for step 2).  There is no
Python or CPU fallback: importing this module without the built library raises ImportError,
and creating a plan without a CUDA device raises BnfftError(BNFFT_E_CUDA).

Functions with the C names (bnfft_plan_create, bnfft_set_nodes, ...) return the raw status
code; `Plan` wraps them for torch tensors (device memory, the current CUDA stream).
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int32, c_int64, c_uint32, c_void_p

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libbnfft.so")
if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_2502_07155_b200.build` "
                      "(there is no CPU fallback)")
_lib = ctypes.CDLL(LIB_PATH)

# ----------------------------------------------------------------------------- constants
BNFFT_OK = 0
STATUS = {
    0: "BNFFT_OK", -1: "BNFFT_E_BAD_DIM", -2: "BNFFT_E_BAD_BANDWIDTH", -3: "BNFFT_E_BAD_SIGMA",
    -4: "BNFFT_E_TRUNCATION_TOO_LARGE", -5: "BNFFT_E_BAD_WINDOW_PARAM",
    -6: "BNFFT_E_SPECTRAL_FACTOR_VANISHES", -7: "BNFFT_E_NODE_NOT_FINITE",
    -8: "BNFFT_E_NODE_OUT_OF_RANGE", -9: "BNFFT_E_NODE_OUTSIDE_FEASIBLE_BOX",
    -10: "BNFFT_E_NODES_NOT_SET", -11: "BNFFT_E_CUDA", -12: "BNFFT_E_CUFFT", -13: "BNFFT_E_OOM",
    -14: "BNFFT_E_UNSUPPORTED", -15: "BNFFT_E_INVALID_ARG", -16: "BNFFT_E_NCCL",
}
globals().update({v: k for k, v in STATUS.items()})
BNFFT_SINH, BNFFT_GAUSS, BNFFT_CKB = 0, 1, 2
BNFFT_C64, BNFFT_C128 = 0, 1
BNFFT_STRICT_DOMAIN = 1
BNFFT_TIMING = 8
BNFFT_EXACT_TAPS = 16
BNFFT_ALG1 = 32
BNFFT_PRECOMPUTE_PSI = 64
BNFFT_SORTED_OUTPUT = 128
BNFFT_BALANCED_SLABS = 256
BNFFT_DIST_REPLICATE, BNFFT_DIST_SLAB = 0, 1
DISTS = {"replicate": BNFFT_DIST_REPLICATE, "slab": BNFFT_DIST_SLAB}
WINDOWS = {"sinh": BNFFT_SINH, "gauss": BNFFT_GAUSS, "ckb": BNFFT_CKB}
PRECS = {"c64": BNFFT_C64, "c128": BNFFT_C128}


class bnfft_opts(ctypes.Structure):
    _fields_ = [("d", c_int32), ("M", c_int64), ("sigma", c_double), ("m", c_int32),
                ("window", c_int32), ("shape", c_double), ("prec", c_int32), ("batch", c_int32),
                ("flags", c_uint32), ("device", c_int32), ("stream", c_void_p),
                ("rank", c_int32), ("nranks", c_int32), ("nccl_comm", c_void_p), ("local_group", c_void_p),
                ("dist", c_int32)]


class bnfft_info(ctypes.Structure):
    _fields_ = [("d", c_int32), ("M", c_int64), ("L", c_int64), ("m", c_int32),
                ("window", c_int32), ("shape", c_double), ("prec", c_int32), ("batch", c_int32),
                ("bin_log2", c_int32 * 3), ("bins_per_dim", c_int64 * 3), ("nbins", c_int64),
                ("user_block_log2", c_int32), ("nkeys", c_int64), ("tap_poly", c_int32),
                ("tap_fit_err", c_double), ("key_bits", c_int32), ("sort_passes", c_int32), ("flatness", c_double),
                ("n_nodes", c_int64), ("grid_bytes", c_int64), ("device_bytes", c_int64),
                ("gather_kernel", c_int32), ("rank", c_int32), ("nranks", c_int32), ("dist", c_int32),
                ("slab_lo", c_int64), ("slab_hi", c_int64), ("n_owned", c_int64), ("halo_bytes", c_int64), ("key_col_bits", c_int32)]


GATHER_KERNELS = {0: "bnfft::gather1_kernel", 1: "bnfft::gather1b_kernel", 2: "bnfft::gather_kernel",
                  3: "bnfft::gatherN_kernel", 4: "bnfft::gather3c_kernel", 5: "bnfft::gather1_kernel",
                  6: "bnfft::gather3s_kernel", 7: "bnfft::gather3y_kernel",
                  8: "bnfft::gather3q_kernel", 9: "bnfft::gather2c_kernel"}


class bnfft_timing(ctypes.Structure):
    _fields_ = [("ms_psihat", c_double), ("ms_keys", c_double), ("ms_sort", c_double),
                ("ms_build", c_double), ("ms_deconv", c_double), ("ms_fft", c_double),
                ("ms_gather", c_double), ("n_psihat", c_int64), ("n_set_nodes", c_int64),
                ("n_execute", c_int64), ("kernel_launches", c_int64), ("ms_exchange", c_double)]


class bnfft_peaks(ctypes.Structure):
    _fields_ = [("sms", c_int32)] + [(f"{k}_{s}", c_double) for k in
                                      ("ffma", "ffma2", "dfma", "ex2", "rsqrt", "rcp", "lds64", "lds128")
                                      for s in ("per_sm_clk", "per_s", "mhz")]


_P = c_void_p
_sig = {
    "bnfft_measure_peaks": (c_int, [c_int32, POINTER(bnfft_peaks)]),
    "bnfft_plan_create": (c_int, [POINTER(bnfft_opts), POINTER(c_void_p)]),
    "bnfft_precompute": (c_int, [_P]),
    "bnfft_set_nodes": (c_int, [_P, c_int64, c_void_p, POINTER(c_int64)]),
    "bnfft_execute": (c_int, [_P, c_void_p, c_void_p]),
    "bnfft_transform": (c_int, [_P, c_int64, c_void_p, c_void_p, c_void_p, POINTER(c_int64)]),
    "bnfft_transform_host": (c_int, [_P, c_int64, c_void_p, c_void_p, c_void_p, POINTER(c_int64)]),
    "bnfft_transform_host_many": (c_int, [_P, c_int32, c_int64, POINTER(c_void_p), POINTER(c_void_p),
                                          POINTER(c_void_p), POINTER(c_int64)]),
    "bnfft_interpolate": (c_int, [_P, c_void_p, c_void_p]),
    "bnfft_kernel_hat": (c_int, [_P, c_int64, c_void_p, c_void_p]),
    "bnfft_get_info": (c_int, [_P, POINTER(bnfft_info)]),
    "bnfft_get_timing": (c_int, [_P, POINTER(bnfft_timing)]),
    "bnfft_reset_timing": (c_int, [_P]),
    "bnfft_get_psihat": (c_int, [_P, c_void_p]),
    "bnfft_get_grid": (c_int, [_P, c_void_p]),
    "bnfft_get_perm": (c_int, [_P, c_void_p]),
    "bnfft_get_bin_offsets": (c_int, [_P, c_void_p]),
    "bnfft_destroy": (c_int, [_P]),
    "bnfft_nccl_unique_id": (c_int, [c_void_p]),
    "bnfft_nccl_comm_init": (c_int, [c_void_p, c_int32, c_int32, c_int32, POINTER(c_void_p)]),
    "bnfft_nccl_comm_destroy": (c_int, [c_void_p]),
    "bnfft_nccl_selftest": (c_int, [c_void_p, c_int64, c_void_p]),
    "bnfft_group_create": (c_int, [c_int32, POINTER(c_void_p)]),
    "bnfft_group_destroy": (c_int, [c_void_p]),
    "bnfft_slab_cuts": (c_int, [c_void_p, c_int64, c_int32, c_int32, c_void_p]),
    "bnfft_slab_owner": (c_int32, [c_void_p, c_int32, c_int64]),
    "bnfft_halo_ranges": (c_int, [c_void_p, c_int32, c_int32, c_int32, c_int64, POINTER(c_int64), POINTER(c_int64)]),
    "bnfft_status_string": (c_char_p, [c_int]),
    "bnfft_last_error": (c_char_p, []),
    "bnfft_build_info": (c_char_p, []),
}
EXPORTED = tuple(_sig)
for _name, (_res, _args) in _sig.items():
    _f = getattr(_lib, _name)
    _f.restype = _res
    _f.argtypes = _args
    globals()[_name] = _f


class BnfftError(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        detail = _lib.bnfft_last_error().decode(errors="replace")
        super().__init__(f"{what}: {STATUS.get(code, code)} ({detail})")


def check(code: int, what: str = "") -> None:
    if code != BNFFT_OK:
        raise BnfftError(code, what)


def _ptr(t) -> int:
    return 0 if t is None else (t if isinstance(t, int) else t.data_ptr())


class Plan:
    """Owning handle of a bnfft plan on one CUDA device (torch tensors for buffers)."""

    def __init__(self, d: int, M: int, sigma: float, m: int, window: str = "sinh",
                 prec: str = "c128", batch: int = 1, shape: float = 0.0, strict: bool = False,
                 timing: bool = False, exact_taps: bool = False, alg1: bool = False,
                 precompute_psi: bool = False, sorted_output: bool = False, device: int = 0,
                 stream: int | None = None, rank: int = 0, nranks: int = 1, nccl_comm: int | None = None,
                 local_group: int | None = None, dist: str = "replicate", balanced_slabs: bool = False):
        import torch
        self._torch = torch
        if stream is None:
            with torch.cuda.device(device):
                stream = torch.cuda.current_stream(device).cuda_stream
        o = bnfft_opts(d=d, M=M, sigma=sigma, m=m, window=WINDOWS[window], shape=shape,
                       prec=PRECS[prec], batch=batch,
                       flags=(BNFFT_STRICT_DOMAIN if strict else 0) | (BNFFT_TIMING if timing else 0)
                       | (BNFFT_EXACT_TAPS if exact_taps else 0) | (BNFFT_ALG1 if alg1 else 0)
                       | (BNFFT_PRECOMPUTE_PSI if precompute_psi else 0)
                       | (BNFFT_SORTED_OUTPUT if sorted_output else 0)
                       | (BNFFT_BALANCED_SLABS if balanced_slabs else 0),
                       device=device, stream=stream, rank=rank, nranks=nranks, nccl_comm=nccl_comm,
                       local_group=local_group, dist=DISTS[dist])
        h = c_void_p()
        check(bnfft_plan_create(ctypes.byref(o), ctypes.byref(h)), "bnfft_plan_create")
        self.h = h
        self.d, self.M, self.m, self.batch, self.prec, self.device = d, M, m, batch, prec, device
        self.cdtype = torch.complex128 if prec == "c128" else torch.complex64
        self.n = 0
        self.n_user = 0
        self.slab = nranks > 1 and dist == "slab"

    # -- C calls
    def precompute(self) -> None:
        check(bnfft_precompute(self.h), "bnfft_precompute")

    def set_nodes(self, x) -> None:
        t = self._torch
        assert x.dtype == t.float64 and x.is_cuda and x.is_contiguous()
        n = x.shape[0]
        bad = c_int64(-1)
        code = bnfft_set_nodes(self.h, n, _ptr(x) if n else None, ctypes.byref(bad))
        if code != BNFFT_OK:
            err = BnfftError(code, "bnfft_set_nodes")
            err.first_bad = bad.value
            raise err
        self.n_user = n
        self.n = n

    def _check_out(self, out):
        # the kernels write batch x n complex values of the plan's precision into `out`
        n_out = self.n_user if self.slab else self.n
        if out.dtype != self.cdtype or not out.is_cuda or out.device.index != self.device \
                or not out.is_contiguous() or out.numel() < self.batch * n_out:
            raise ValueError("out must be a contiguous CUDA tensor of dtype %s on cuda:%d with >= %d "
                             "elements" % (self.cdtype, self.device, self.batch * n_out))

    def execute(self, fhat, out=None):
        t = self._torch
        assert fhat.dtype == self.cdtype and fhat.is_cuda and fhat.is_contiguous()
        assert fhat.numel() == self.batch * self.M ** self.d
        if out is None:
            out = t.empty((self.batch, self.n), dtype=self.cdtype, device=fhat.device)
        self._check_out(out)
        check(bnfft_execute(self.h, _ptr(fhat), _ptr(out) if (self.n or self.slab) else None), "bnfft_execute")
        return out

    def transform(self, x, fhat, out=None):
        """Algorithm 2 in one call (bnfft_transform): the grid stage overlaps the node sort."""
        t = self._torch
        assert x.dtype == t.float64 and x.is_cuda and x.is_contiguous()
        assert fhat.dtype == self.cdtype and fhat.is_cuda and fhat.is_contiguous()
        assert fhat.numel() == self.batch * self.M ** self.d
        n = x.shape[0]
        if out is None:
            out = t.empty((self.batch, n), dtype=self.cdtype, device=fhat.device)
        self.n_user = n
        self.n = n
        self._check_out(out)
        bad = c_int64(-1)
        code = bnfft_transform(self.h, n, _ptr(x) if n else None, _ptr(fhat),
                               _ptr(out) if (n or self.slab) else None, ctypes.byref(bad))
        if code != BNFFT_OK:
            err = BnfftError(code, "bnfft_transform")
            err.first_bad = bad.value
            raise err
        return out

    def interpolate(self, samples, out=None):
        """Step 3 alone from grid samples (batch x L^d, centred): regularized Shannon formula."""
        t = self._torch
        assert samples.dtype == self.cdtype and samples.is_cuda and samples.is_contiguous()
        if out is None:
            out = t.empty((self.batch, self.n), dtype=self.cdtype, device=samples.device)
        self._check_out(out)
        check(bnfft_interpolate(self.h, _ptr(samples), _ptr(out) if self.n else None), "bnfft_interpolate")
        return out

    def kernel_hat(self, v):
        import numpy as np
        v = np.ascontiguousarray(v, dtype=np.float64)
        out = np.empty_like(v)
        check(bnfft_kernel_hat(self.h, v.size, v.ctypes.data, out.ctypes.data), "bnfft_kernel_hat")
        return out

    def transform_host(self, x_host, fhat_host, f_host) -> None:
        bad = c_int64(-1)
        check(bnfft_transform_host(self.h, x_host.shape[0], _ptr(x_host), _ptr(fhat_host),
                                   _ptr(f_host), ctypes.byref(bad)), "bnfft_transform_host")

    def transform_host_many(self, xs, fhats, fs) -> None:
        """Pipelined host transforms (bnfft_transform_host_many): step k reads xs[k], fhats[k] and
        writes fs[k] (pinned host tensors; consecutive outputs must be distinct buffers)."""
        k = len(xs)
        assert len(fhats) == k and len(fs) == k
        n = xs[0].shape[0] if k else 0
        arr = c_void_p * max(k, 1)
        bad = c_int64(-1)
        code = bnfft_transform_host_many(self.h, k, n, arr(*[_ptr(t) for t in xs]), arr(*[_ptr(t) for t in fhats]),
                                         arr(*[_ptr(t) for t in fs]), ctypes.byref(bad))
        if code != BNFFT_OK:
            err = BnfftError(code, "bnfft_transform_host_many")
            err.first_bad = bad.value
            raise err

    def info(self) -> bnfft_info:
        i = bnfft_info()
        check(bnfft_get_info(self.h, ctypes.byref(i)), "bnfft_get_info")
        return i

    def timing(self) -> bnfft_timing:
        tm = bnfft_timing()
        check(bnfft_get_timing(self.h, ctypes.byref(tm)), "bnfft_get_timing")
        return tm

    def reset_timing(self) -> None:
        check(bnfft_reset_timing(self.h), "bnfft_reset_timing")

    def psihat(self):
        import numpy as np
        a = np.empty(self.M, dtype=np.float64)
        check(bnfft_get_psihat(self.h, a.ctypes.data), "bnfft_get_psihat")
        return a

    def grid(self):
        t = self._torch
        i = self.info()
        g = t.empty((self.batch,) + (i.L,) * self.d, dtype=self.cdtype, device=f"cuda:{self.device}")
        check(bnfft_get_grid(self.h, _ptr(g)), "bnfft_get_grid")
        return g

    def perm(self):
        t = self._torch
        p = t.empty(max(self.n, 1), dtype=t.int32, device=f"cuda:{self.device}")
        check(bnfft_get_perm(self.h, _ptr(p)), "bnfft_get_perm")
        return p[: self.n]

    def bin_offsets(self):
        t = self._torch
        i = self.info()
        o = t.empty(i.nkeys + 1, dtype=t.int32, device=f"cuda:{self.device}")
        check(bnfft_get_bin_offsets(self.h, _ptr(o)), "bnfft_get_bin_offsets")
        return o

    def close(self) -> None:
        if getattr(self, "h", None):
            bnfft_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def measure_peaks(device: int = 0) -> dict:
    """Pipe-throughput microbenchmarks (bnfft_measure_peaks) as a dict."""
    pk = bnfft_peaks()
    check(bnfft_measure_peaks(device, ctypes.byref(pk)), "bnfft_measure_peaks")
    return {f: getattr(pk, f) for f, _ in bnfft_peaks._fields_}


# ----------------------------------------------------------------------------- multi-GPU helpers
def slab_cuts(L: int, nranks: int, align: int, plane_counts=None):
    """Cut points of BNFFT_DIST_SLAB (bnfft_slab_cuts): equal planes, or balanced by plane_counts."""
    import numpy as np
    cuts = np.zeros(nranks + 1, dtype=np.int64)
    pc = None if plane_counts is None else np.ascontiguousarray(plane_counts, dtype=np.int64)
    check(bnfft_slab_cuts(None if pc is None else pc.ctypes.data, L, nranks, align, cuts.ctypes.data),
          "bnfft_slab_cuts")
    return cuts


def slab_owner(cuts, c: int) -> int:
    import numpy as np
    cuts = np.ascontiguousarray(cuts, dtype=np.int64)
    return int(bnfft_slab_owner(cuts.ctypes.data, len(cuts) - 1, c))


def halo_ranges(cuts, rank: int, m: int, L: int):
    import numpy as np
    cuts = np.ascontiguousarray(cuts, dtype=np.int64)
    lo, hi = c_int64(), c_int64()
    check(bnfft_halo_ranges(cuts.ctypes.data, len(cuts) - 1, rank, m, L, ctypes.byref(lo), ctypes.byref(hi)),
          "bnfft_halo_ranges")
    return lo.value, hi.value


class Group:
    """In-process transport of nranks plans (bnfft_group_create); each rank runs in its own thread."""

    def __init__(self, nranks: int):
        h = c_void_p()
        check(bnfft_group_create(nranks, ctypes.byref(h)), "bnfft_group_create")
        self.h = h
        self.nranks = nranks

    @property
    def handle(self) -> int:
        return self.h.value

    def close(self):
        if self.h:
            bnfft_group_destroy(self.h)
            self.h = None


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    check(bnfft_nccl_unique_id(buf), "bnfft_nccl_unique_id")
    return buf.raw


def nccl_comm_init(uid: bytes, nranks: int, rank: int, device: int) -> int:
    h = c_void_p()
    buf = ctypes.create_string_buffer(uid, 128)
    check(bnfft_nccl_comm_init(buf, nranks, rank, device, ctypes.byref(h)), "bnfft_nccl_comm_init")
    return h.value


def nccl_selftest(comm: int, nbytes: int = 1 << 20, stream: int = 0) -> None:
    """Collective check of the library's NCCL transport (bnfft_nccl_selftest); raises on failure."""
    check(bnfft_nccl_selftest(comm, nbytes, stream), "bnfft_nccl_selftest")


def nccl_comm_destroy(comm: int) -> None:
    check(bnfft_nccl_comm_destroy(comm), "bnfft_nccl_comm_destroy")


def torch_nccl_comm(group=None, device=None) -> int:
    """The ncclComm_t of torch.distributed's NCCL process group (ProcessGroupNCCL._comm_ptr)."""
    import torch
    import torch.distributed as dist
    pg = group or dist.distributed_c10d._get_default_group()
    dev = device or torch.device("cuda", torch.cuda.current_device())
    return int(pg._get_backend(dev)._comm_ptr())
