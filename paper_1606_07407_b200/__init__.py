"""paper_1606_07407_b200 -- B200-native multidimensional phase-shift sparse FFT (arXiv 1606.07407).

Thin ctypes binding over ``libsfft.so`` (include/sfft.h).  The functions carry the C names
and only marshal arguments: every step of Algorithm 2 runs in the library's sm_100a kernels.
PyTorch supplies device memory (the plan workspace and the output tensors), the current CUDA
stream and, for multi-GPU runs, ``torch.distributed``.  There is no CPU fallback: if the
library or a CUDA device is missing, the calls raise.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass
from typing import Optional, Sequence, Tuple

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SFFT_LIB_PATH") or os.path.join(_HERE, "libsfft.so")   # env: tuning builds only

SFFT_OK, SFFT_PARTIAL = 0, 1
SFFT_EINVAL, SFFT_EPRECISION, SFFT_EDIM, SFFT_ECORRUPT = -1, -2, -3, -4
SFFT_ECUDA, SFFT_ENOMEM, SFFT_ENCCL, SFFT_ENOTSUP = -5, -6, -7, -8

# every symbol include/sfft.h declares (checked by tests/test_abi.py)
EXPORTS = (
    "sfft_plan", "sfft_plan_workspace_size", "sfft_plan_set_workspace", "sfft_plan_info",
    "sfft_plan_destroy", "sfft_signal_expsum", "sfft_signal_destroy", "sfft_execute",
    "sfft_solve_host", "sfft_solve_host_batches", "sfft_stage_expsum", "sfft_stage_pfft", "sfft_stage_decode",
    "sfft_stage_project", "sfft_comm_init", "sfft_comm_unique_id", "sfft_execute_group",
    "sfft_line_shard_range", "sfft_comm_peer_handle", "sfft_comm_init_peers", "sfft_strerror",
    "sfft_last_error", "sfft_version",
)


class sfft_tilt(ctypes.Structure):
    _fields_ = [("axis0", ctypes.c_int32), ("axis1", ctypes.c_int32),
                ("base", ctypes.c_int64), ("height", ctypes.c_int64), ("hypo", ctypes.c_int64)]


class sfft_options(ctypes.Structure):
    _fields_ = [("n_blocks", ctypes.c_int32), ("block_dims", ctypes.POINTER(ctypes.c_int32)),
                ("c", ctypes.c_int32), ("tol", ctypes.c_double), ("bin_floor_rel", ctypes.c_double),
                ("prune_floor", ctypes.c_double), ("round_tol", ctypes.c_double),
                ("max_iter", ctypes.c_int32), ("stall_limit", ctypes.c_int32),
                ("batch", ctypes.c_int32), ("extra_checks", ctypes.c_int32),
                ("stream", ctypes.c_void_p), ("profile", ctypes.c_int32),
                ("literal_residual", ctypes.c_int32), ("expsum_path", ctypes.c_int32),
                ("fallback_tilts", ctypes.c_int32), ("line_shards", ctypes.c_int32),
                ("line_rank", ctypes.c_int32), ("table_cache_slots", ctypes.c_int32),
                ("line_exchange", ctypes.c_int32), ("spec_primes", ctypes.c_int32),
                ("spec_distributed", ctypes.c_int32), ("spec_rank", ctypes.c_int32)]


class sfft_report(ctypes.Structure):
    _fields_ = [("samples_used", ctypes.c_int64), ("cmacs", ctypes.c_int64),
                ("iterations", ctypes.c_int32), ("n_ok", ctypes.c_int32),
                ("n_partial", ctypes.c_int32), ("n_error", ctypes.c_int32),
                ("status", ctypes.c_int32), ("n_iter_logged", ctypes.c_int32),
                ("primes", ctypes.c_int64 * 64), ("accepted", ctypes.c_int32 * 64),
                ("kernel_launches", ctypes.c_int32), ("n_expsum", ctypes.c_int32),
                ("ms_expsum", ctypes.c_float), ("ms_fft", ctypes.c_float), ("ms_decode", ctypes.c_float),
                ("ms_other", ctypes.c_float), ("i8_limbs", ctypes.c_int32), ("n_expsum_i8", ctypes.c_int32),
                ("cmacs_i8", ctypes.c_int64), ("ms_expsum_i8", ctypes.c_float),
                ("fallback_used", ctypes.c_int32), ("ms_total", ctypes.c_float), ("fft_plogp", ctypes.c_double),
                ("fft_mlogm", ctypes.c_double), ("n_fused_sample", ctypes.c_int32)]


class SfftError(RuntimeError):
    def __init__(self, status: int, msg: str = ""):
        super().__init__(f"sfft status {status} ({strerror(status)}) {msg}".strip())
        self.status = status


_lib = None


def lib() -> ctypes.CDLL:
    """Load libsfft.so (built in-tree by __graft_entry__.build()); raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
                              " (there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        vp, i32, i64, dbl = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_double
        L.sfft_plan.argtypes = [i32, i64, i32, vp, i32, vp, i32, dbl, vp, ctypes.POINTER(vp)]
        L.sfft_plan_workspace_size.argtypes = [vp, ctypes.POINTER(ctypes.c_size_t)]
        L.sfft_plan_set_workspace.argtypes = [vp, vp, ctypes.c_size_t]
        L.sfft_plan_info.argtypes = [vp, vp, vp, vp, vp, vp]
        L.sfft_plan_destroy.argtypes = [vp]
        L.sfft_plan_destroy.restype = None
        L.sfft_signal_expsum.argtypes = [vp, i32, vp, vp, ctypes.POINTER(vp)]
        L.sfft_signal_destroy.argtypes = [vp]
        L.sfft_signal_destroy.restype = None
        L.sfft_execute.argtypes = [vp, vp, vp, vp, vp, vp, vp]
        L.sfft_solve_host.argtypes = [vp, i32, vp, vp, vp, vp, vp, vp, vp]
        L.sfft_solve_host_batches.argtypes = [vp, i32, i32, vp, vp, vp, vp, vp, vp, vp]
        L.sfft_stage_expsum.argtypes = [vp, i32, vp, vp, i64, i32, vp]
        L.sfft_stage_pfft.argtypes = [vp, i32, i64, vp]
        L.sfft_stage_decode.argtypes = [vp, i64, i32, i32, vp, vp, vp, vp, vp]
        L.sfft_stage_project.argtypes = [vp, vp, vp]
        L.sfft_comm_init.argtypes = [vp, i32, i32, vp, i32]
        L.sfft_comm_unique_id.argtypes = [vp]
        L.sfft_comm_peer_handle.argtypes = [vp, vp]
        L.sfft_comm_init_peers.argtypes = [vp, i32, i32, vp]
        L.sfft_line_shard_range.argtypes = [i32, i32, i32, vp, vp]
        L.sfft_execute_group.argtypes = [vp, vp, i32, vp, vp, vp, vp, vp]
        L.sfft_strerror.argtypes = [ctypes.c_int]
        L.sfft_strerror.restype = ctypes.c_char_p
        L.sfft_last_error.argtypes = [vp]
        L.sfft_last_error.restype = ctypes.c_char_p
        L.sfft_version.argtypes = []
        L.sfft_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


def strerror(status: int) -> str:
    try:
        return lib().sfft_strerror(status).decode()
    except ImportError:
        return "?"


def sfft_version() -> str:
    return lib().sfft_version().decode()


def _torch():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_1606_07407_b200 needs a CUDA device (no CPU fallback)")
    return torch


def _ptr(t) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _check(rc: int, plan=None, ok=(SFFT_OK,)):
    if rc not in ok:
        msg = ""
        if plan is not None:
            msg = lib().sfft_last_error(plan).decode()
        raise SfftError(rc, msg)
    return rc


class Plan:
    """Owns an sfft_plan_t and its torch-allocated workspace (sfft_plan / sfft_plan_set_workspace)."""

    def __init__(self, handle, workspace, d, N, k, batch, opts_keep):
        self.handle = handle
        self.workspace = workspace
        self.d, self.N, self.k, self.batch = d, N, k, batch
        self._keep = opts_keep
        E, r, L, pmax, tn = (ctypes.c_int64(), ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64(),
                             ctypes.c_int32())
        lib().sfft_plan_info(handle, ctypes.byref(E), ctypes.byref(r), ctypes.byref(L), ctypes.byref(pmax),
                             ctypes.byref(tn))
        self.E, self.r, self.L, self.p_max, self.tile_n = E.value, r.value, L.value, pmax.value, tn.value

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                lib().sfft_plan_destroy(h)
            except Exception:
                pass
            self.handle = None


def sfft_plan(d: int, N: int, k: int, primes: Optional[Sequence[int]] = None,
              tilts: Sequence[Tuple[int, int, int, int, int]] = (), eps: float = 0.0,
              blocks: Optional[Sequence[int]] = None, batch: int = 1, c: int = 5, tol: float = 1e-6,
              bin_floor_rel: float = 1e-8, prune_floor: float = 1e-8, round_tol: float = 0.01,
              max_iter: int = 1000, stall_limit: int = 0, extra_checks: int = 3,
              stream=None, profile: bool = False, literal_residual: bool = False,
              expsum_path: int = 0, fallback_tilts: int = 0, line_shards: int = 0, line_rank: int = 0,
              table_cache_slots: int = 0, line_exchange: int = 0, spec_primes: int = 0,
              spec_distributed: int = 0, spec_rank: int = 0) -> Plan:
    """sfft_plan(d, N, k, primes, tilts, eps) of include/sfft.h; workspace from torch on the current device."""
    torch = _torch()
    L = lib()
    keep = []
    opt = sfft_options()
    if blocks is not None:
        arr = (ctypes.c_int32 * len(blocks))(*blocks)
        keep.append(arr)
        opt.n_blocks, opt.block_dims = len(blocks), ctypes.cast(arr, ctypes.POINTER(ctypes.c_int32))
    opt.c, opt.tol, opt.bin_floor_rel, opt.prune_floor, opt.round_tol = c, tol, bin_floor_rel, prune_floor, round_tol
    opt.max_iter, opt.stall_limit, opt.batch, opt.extra_checks = max_iter, stall_limit, batch, extra_checks
    st = stream if stream is not None else torch.cuda.current_stream()
    opt.stream = ctypes.c_void_p(st.cuda_stream)
    opt.profile = 1 if profile else 0
    opt.literal_residual = 1 if literal_residual else 0
    opt.expsum_path = int(expsum_path)
    opt.fallback_tilts = int(fallback_tilts)
    opt.line_shards, opt.line_rank = int(line_shards), int(line_rank)
    opt.table_cache_slots = int(table_cache_slots)
    opt.line_exchange = int(line_exchange)
    opt.spec_primes = int(spec_primes)
    opt.spec_distributed, opt.spec_rank = int(spec_distributed), int(spec_rank)
    pr = None
    if primes is not None:
        pr = (ctypes.c_int64 * len(primes))(*primes)
        keep.append(pr)
    tl = None
    if tilts:
        tl = (sfft_tilt * len(tilts))(*[sfft_tilt(*t) for t in tilts])
        keep.append(tl)
    h = ctypes.c_void_p()
    rc = L.sfft_plan(d, N, k, ctypes.cast(pr, ctypes.c_void_p) if pr is not None else None,
                     len(primes) if primes is not None else 0,
                     ctypes.cast(tl, ctypes.c_void_p) if tl is not None else None, len(tilts), eps,
                     ctypes.byref(opt), ctypes.byref(h))
    _check(rc)
    nb = ctypes.c_size_t()
    L.sfft_plan_workspace_size(h, ctypes.byref(nb))
    ws = torch.empty(nb.value, dtype=torch.uint8, device="cuda")
    _check(L.sfft_plan_set_workspace(h, ctypes.c_void_p(ws.data_ptr()), nb.value), h)
    keep.append(opt)
    return Plan(h, ws, d, N, k, batch, keep)


class Signal:
    def __init__(self, handle, freqs, coeffs_f64, batch):
        self.handle, self.freqs, self.coeffs, self.batch = handle, freqs, coeffs_f64, batch

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                lib().sfft_signal_destroy(h)
            except Exception:
                pass
            self.handle = None


def _coeff_view(coeffs):
    torch = _torch()
    if coeffs.is_complex():
        coeffs = torch.view_as_real(coeffs)
    return coeffs.contiguous()


def _require(t, name: str, shape, dtype, cuda: bool = True, pinned_ok: bool = True):
    """Argument check of the binding (the C ABI only sees raw pointers): raises ValueError, never asserts."""
    if t is None:
        raise ValueError(f"{name}: missing")
    if tuple(t.shape) != tuple(shape):
        raise ValueError(f"{name}: shape {tuple(t.shape)}, expected {tuple(shape)}")
    if t.dtype != dtype:
        raise ValueError(f"{name}: dtype {t.dtype}, expected {dtype}")
    if cuda and not t.is_cuda:
        raise ValueError(f"{name}: must be a CUDA tensor")
    if not cuda and t.is_cuda:
        raise ValueError(f"{name}: must be a host tensor")
    if not t.is_contiguous():
        raise ValueError(f"{name}: must be contiguous")


def _check_outs(plan, out, B: int, cuda: bool):
    torch = _torch()
    if len(out) != 4:
        raise ValueError("out: expected (freqs, coeffs, count, status)")
    of, oc, on, os_ = out
    _require(of, "out freqs", (B, plan.k, plan.d), torch.int32, cuda)
    if oc is not None and oc.is_complex():
        _require(oc, "out coeffs", (B, plan.k), torch.complex128, cuda)
    else:
        _require(oc, "out coeffs", (B, plan.k, 2), torch.float64, cuda)
    _require(on, "out count", (B,), torch.int32, cuda)
    _require(os_, "out status", (B,), torch.int32, cuda)


def sfft_signal_expsum(plan: Plan, freqs, coeffs) -> Signal:
    """f(t) = sum_j a_j e^{2 pi i omega_j . t}: freqs int32 [B,k,d] and coeffs complex128 [B,k] on the GPU."""
    torch = _torch()
    if freqs.dim() != 3:
        raise ValueError(f"freqs: expected [batch, k, d], got shape {tuple(freqs.shape)}")
    batch = freqs.shape[0]
    if batch < 1 or batch > plan.batch:
        raise ValueError(f"freqs: batch {batch} outside [1, plan batch {plan.batch}]")
    _require(freqs, "freqs", (batch, plan.k, plan.d), torch.int32)
    c = _coeff_view(coeffs)
    _require(c, "coeffs", (batch, plan.k, 2), torch.float64)
    h = ctypes.c_void_p()
    _check(lib().sfft_signal_expsum(plan.handle, batch, ctypes.c_void_p(freqs.data_ptr()),
                                    ctypes.c_void_p(c.data_ptr()), ctypes.byref(h)), plan.handle)
    return Signal(h, freqs, c, batch)


@dataclass
class Result:
    status: int
    freqs: object      # int32 [B,k,d]
    coeffs: object     # complex128 [B,k]
    count: object      # int32 [B]
    per_status: object  # int32 [B]
    report: sfft_report


def sfft_execute(plan: Plan, sig: Signal, out=None) -> Result:
    """Run Algorithm 2 on every signal of the batch (device outputs, canonical order)."""
    torch = _torch()
    B = sig.batch
    if out is None:
        out = (torch.empty((B, plan.k, plan.d), dtype=torch.int32, device="cuda"),
               torch.empty((B, plan.k, 2), dtype=torch.float64, device="cuda"),
               torch.empty((B,), dtype=torch.int32, device="cuda"),
               torch.empty((B,), dtype=torch.int32, device="cuda"))
    _check_outs(plan, out, B, cuda=True)
    of, oc, on, os_ = out
    rep = sfft_report()
    rc = lib().sfft_execute(plan.handle, sig.handle, ctypes.c_void_p(of.data_ptr()), ctypes.c_void_p(oc.data_ptr()),
                            ctypes.c_void_p(on.data_ptr()), ctypes.c_void_p(os_.data_ptr()), ctypes.byref(rep))
    _check(rc, plan.handle, ok=(SFFT_OK, SFFT_PARTIAL, SFFT_ENOTSUP, SFFT_ECORRUPT))
    return Result(rc, of, torch.view_as_complex(oc), on, os_, rep)


def sfft_solve_host(plan: Plan, freqs, coeffs, out=None) -> Result:
    """End-to-end call with HOST tensors (pinned for full speed): H2D, solve, D2H inside the library."""
    torch = _torch()
    if freqs.dim() != 3:
        raise ValueError(f"freqs: expected [batch, k, d], got shape {tuple(freqs.shape)}")
    B = freqs.shape[0]
    if B < 1 or B > plan.batch:
        raise ValueError(f"freqs: batch {B} outside [1, plan batch {plan.batch}]")
    _require(freqs, "freqs", (B, plan.k, plan.d), torch.int32, cuda=False)
    c = coeffs if not coeffs.is_complex() else torch.view_as_real(coeffs)
    _require(c, "coeffs", (B, plan.k, 2), torch.float64, cuda=False)
    if out is None:
        out = (torch.empty((B, plan.k, plan.d), dtype=torch.int32).pin_memory(),
               torch.empty((B, plan.k, 2), dtype=torch.float64).pin_memory(),
               torch.empty((B,), dtype=torch.int32).pin_memory(),
               torch.empty((B,), dtype=torch.int32).pin_memory())
    _check_outs(plan, out, B, cuda=False)
    of, oc, on, os_ = out
    rep = sfft_report()
    rc = lib().sfft_solve_host(plan.handle, B, ctypes.c_void_p(freqs.data_ptr()), ctypes.c_void_p(c.data_ptr()),
                               ctypes.c_void_p(of.data_ptr()), ctypes.c_void_p(oc.data_ptr()),
                               ctypes.c_void_p(on.data_ptr()), ctypes.c_void_p(os_.data_ptr()), ctypes.byref(rep))
    _check(rc, plan.handle, ok=(SFFT_OK, SFFT_PARTIAL, SFFT_ENOTSUP, SFFT_ECORRUPT))
    return Result(rc, of, torch.view_as_complex(oc), on, os_, rep)


def sfft_solve_host_batches(plan: Plan, freqs, coeffs, out=None):
    """n_batches batches of HOST tensors (pinned for the overlap): freqs int32 [n_batches, batch, k, d], coeffs
    complex128 [n_batches, batch, k] (or float64 [..., 2]).  The library overlaps the H2D / D2H of neighbouring
    batches with each solve.  Returns (status, out_freqs, out_coeffs, out_count, out_status, [reports])."""
    torch = _torch()
    if freqs.dim() != 4:
        raise ValueError(f"freqs: expected [n_batches, batch, k, d], got shape {tuple(freqs.shape)}")
    nb, B = freqs.shape[0], freqs.shape[1]
    if nb < 1:
        raise ValueError("freqs: no batches")
    if B < 1 or B > plan.batch:
        raise ValueError(f"freqs: batch {B} outside [1, plan batch {plan.batch}]")
    _require(freqs, "freqs", (nb, B, plan.k, plan.d), torch.int32, cuda=False)
    c = coeffs if not coeffs.is_complex() else torch.view_as_real(coeffs)
    _require(c, "coeffs", (nb, B, plan.k, 2), torch.float64, cuda=False)
    if out is None:
        out = (torch.empty((nb, B, plan.k, plan.d), dtype=torch.int32).pin_memory(),
               torch.empty((nb, B, plan.k, 2), dtype=torch.float64).pin_memory(),
               torch.empty((nb, B), dtype=torch.int32).pin_memory(),
               torch.empty((nb, B), dtype=torch.int32).pin_memory())
    if len(out) != 4:
        raise ValueError("out: expected (freqs, coeffs, count, status)")
    of, oc, on, os_ = out
    oc = oc if not oc.is_complex() else torch.view_as_real(oc)
    _require(of, "out freqs", (nb, B, plan.k, plan.d), torch.int32, cuda=False)
    _require(oc, "out coeffs", (nb, B, plan.k, 2), torch.float64, cuda=False)
    _require(on, "out count", (nb, B), torch.int32, cuda=False)
    if os_ is not None:
        _require(os_, "out status", (nb, B), torch.int32, cuda=False)
    reps = (sfft_report * nb)()
    rc = lib().sfft_solve_host_batches(plan.handle, nb, B, ctypes.c_void_p(freqs.data_ptr()),
                                       ctypes.c_void_p(c.data_ptr()), ctypes.c_void_p(of.data_ptr()),
                                       ctypes.c_void_p(oc.data_ptr()), ctypes.c_void_p(on.data_ptr()),
                                       ctypes.c_void_p(_ptr(os_)), ctypes.cast(reps, ctypes.c_void_p))
    _check(rc, plan.handle, ok=(SFFT_OK, SFFT_PARTIAL, SFFT_ENOTSUP, SFFT_ECORRUPT))
    return rc, of, torch.view_as_complex(oc), on, os_, list(reps)


# ------------------------------------------------------------------ stage entry points
def sfft_stage_expsum(plan: Plan, v, c, p: int, m: int):
    """Lines of one iteration: v int64 [r, K], c complex128 [K] (device) -> complex128 [L, p]."""
    torch = _torch()
    if v.dim() != 2 or v.shape[0] != plan.r:
        raise ValueError(f"v: expected [r={plan.r}, K], got shape {tuple(v.shape)}")
    K = v.shape[1]
    v = v.contiguous()
    _require(v, "v", (plan.r, K), torch.int64)
    cc = _coeff_view(c)
    _require(cc, "c", (K, 2), torch.float64)
    out = torch.empty((plan.L, p, 2), dtype=torch.float64, device="cuda")
    _check(lib().sfft_stage_expsum(plan.handle, K, ctypes.c_void_p(v.data_ptr()), ctypes.c_void_p(cc.data_ptr()),
                                   p, m, ctypes.c_void_p(out.data_ptr())), plan.handle)
    return torch.view_as_complex(out)


def sfft_stage_pfft(plan: Plan, x):
    """In-place DFT of every row of x (complex128 [n_lines, p], device); returns x."""
    torch = _torch()
    if x.dim() != 2 or x.dtype != torch.complex128 or not x.is_cuda or not x.is_contiguous():
        raise ValueError("x: expected a contiguous complex128 CUDA tensor [n_lines, p]")
    xr = torch.view_as_real(x)
    _check(lib().sfft_stage_pfft(plan.handle, x.shape[0], x.shape[1], ctypes.c_void_p(xr.data_ptr())), plan.handle)
    return x


def sfft_stage_decode(plan: Plan, F, p: int, m: int, kstar: int):
    """Select + test + decode of one iteration: F complex128 [L, p] (device).
    Returns (n_candidates, bins int32 [na], v int64 [na, r], a complex128 [na]) on the device."""
    torch = _torch()
    _require(F.contiguous(), "F", (plan.L, p), torch.complex128)
    Fr = torch.view_as_real(F.contiguous())
    acc_b = torch.zeros(kstar, dtype=torch.int32, device="cuda")
    acc_v = torch.zeros((plan.r, kstar), dtype=torch.int64, device="cuda")
    acc_a = torch.zeros((kstar, 2), dtype=torch.float64, device="cuda")
    counts = torch.zeros(2, dtype=torch.int32, device="cuda")
    _check(lib().sfft_stage_decode(plan.handle, p, m, kstar, ctypes.c_void_p(Fr.data_ptr()),
                                   ctypes.c_void_p(acc_b.data_ptr()), ctypes.c_void_p(acc_v.data_ptr()),
                                   ctypes.c_void_p(acc_a.data_ptr()), ctypes.c_void_p(counts.data_ptr())),
           plan.handle)
    nc, na = (int(x) for x in counts.tolist())
    return nc, acc_b[:na], acc_v[:, :na].T.contiguous(), torch.view_as_complex(acc_a[:na].contiguous())


def sfft_stage_project(plan: Plan, sig: Signal):
    """Reduced (tilted) frequencies int64 [B, r, k] of a signal (Eq. (35), Eq. (27))."""
    torch = _torch()
    out = torch.empty((sig.batch, plan.r, plan.k), dtype=torch.int64, device="cuda")
    _check(lib().sfft_stage_project(plan.handle, sig.handle, ctypes.c_void_p(out.data_ptr())), plan.handle)
    return out


def sfft_comm_init(plan: Plan, nranks: int, rank: int, shard_mode: int = 0, unique_id: bytes = b""):
    buf = ctypes.create_string_buffer(unique_id, 128) if unique_id else None
    return _check(lib().sfft_comm_init(plan.handle, nranks, rank, buf, shard_mode), plan.handle)


def sfft_line_shard_range(r: int, G: int, g: int) -> Tuple[int, int]:
    """Reduced axes [lo, hi) of line shard g of G (host call, no device needed)."""
    lo, hi = ctypes.c_int32(), ctypes.c_int32()
    _check(lib().sfft_line_shard_range(r, G, g, ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def sfft_comm_unique_id() -> bytes:
    """128-byte NCCL unique id (rank 0 of a line-sharded job; broadcast it with torch.distributed)."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().sfft_comm_unique_id(buf))
    return buf.raw


def sfft_execute_group(plans: Sequence[Plan], sigs: Sequence[Signal], out=None) -> Result:
    """Line-sharded solve of len(plans) shards, or the ranks of a distributed speculation (spec_distributed plans),
    on ONE device (include/sfft.h sfft_execute_group)."""
    torch = _torch()
    n = len(plans)
    B, p0 = sigs[0].batch, plans[0]
    if out is None:
        out = (torch.empty((B, p0.k, p0.d), dtype=torch.int32, device="cuda"),
               torch.empty((B, p0.k, 2), dtype=torch.float64, device="cuda"),
               torch.empty((B,), dtype=torch.int32, device="cuda"),
               torch.empty((B,), dtype=torch.int32, device="cuda"))
    of, oc, on, os_ = out
    hp = (ctypes.c_void_p * n)(*[p.handle for p in plans])
    hs = (ctypes.c_void_p * n)(*[s.handle for s in sigs])
    rep = sfft_report()
    rc = lib().sfft_execute_group(hp, hs, n, ctypes.c_void_p(of.data_ptr()), ctypes.c_void_p(oc.data_ptr()),
                                  ctypes.c_void_p(on.data_ptr()), ctypes.c_void_p(os_.data_ptr()), ctypes.byref(rep))
    _check(rc, p0.handle, ok=(SFFT_OK, SFFT_PARTIAL, SFFT_ENOTSUP))
    return Result(rc, of, torch.view_as_complex(oc), on, os_, rep)


def sfft_comm_peer_handle(plan: Plan) -> bytes:
    """64-byte CUDA IPC handle of this shard's record-exchange buffer (plans with line_exchange = 1)."""
    buf = ctypes.create_string_buffer(64)
    _check(lib().sfft_comm_peer_handle(plan.handle, buf), plan.handle)
    return buf.raw


def sfft_comm_init_peers(plan: Plan, nranks: int, rank: int, handles: Sequence[bytes]) -> int:
    """Open the other shards' exchange buffers (collective over the line shards; handles of all ranks in rank
    order, 64 bytes each)."""
    if len(handles) != nranks or any(len(h) != 64 for h in handles):
        raise ValueError("handles: one 64-byte handle per rank")
    blob = ctypes.create_string_buffer(b"".join(handles), 64 * nranks)
    return _check(lib().sfft_comm_init_peers(plan.handle, nranks, rank, blob), plan.handle)


def exchange_handles(local: bytes, group=None) -> list:
    """All-gather one opaque byte string per rank over a torch.distributed group (CPU-testable with gloo)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, local, group=group)
    return out


def comm_init_spec_ranks(plan: Plan, group=None) -> None:
    """Distributed multi-prime speculation (R26) over a torch.distributed group: rank 0 draws the NCCL id, the group
    broadcasts it, every rank initialises the plan's communicator (shard_mode 2, collective)."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [sfft_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    sfft_comm_init(plan, world, rank, shard_mode=2, unique_id=obj[0])


def comm_init_line_shards(plan: Plan, group=None, exchange: int = 0) -> None:
    """Line sharding over a torch.distributed group.  exchange 0: rank 0 draws the NCCL id, the group broadcasts it
    (broadcast_object_list), every rank initialises the plan's communicator (collective).  exchange 1 (plans with
    line_exchange = 1): the ranks all-gather the CUDA IPC handles of their exchange buffers and open each other's,
    so the FFT epilogue stores the records into every shard's memory directly."""
    import torch.distributed as dist
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if exchange == 1:
        sfft_comm_init_peers(plan, world, rank, exchange_handles(sfft_comm_peer_handle(plan), group))
        return
    obj = [sfft_comm_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    sfft_comm_init(plan, world, rank, shard_mode=1, unique_id=obj[0])


def solve(plan: Plan, freqs, coeffs):
    """Convenience: device tensors in, Result out (one sfft_signal_expsum + sfft_execute)."""
    sig = sfft_signal_expsum(plan, freqs, coeffs)
    return sfft_execute(plan, sig)
