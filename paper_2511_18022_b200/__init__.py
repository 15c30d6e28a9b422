"""paper_2511_18022_b200 -- B200-native scenario-parallel Split DP (arXiv 2511.18022).

Thin Python binding over the C-ABI library ``libspdp.so`` (declared in
``include/spdp.h``): argument marshalling only.  Every step of the hot path
runs in the CUDA kernels of ``csrc/``; PyTorch supplies device memory, the
current stream and (in ``dist``) process groups.  There is no CPU fallback:
importing this package without the built library raises ImportError, and
calling a kernel entry point without a CUDA device raises SpdpError.

Names follow the paper: ``split_eval`` evaluates Eq. (1)-(3)
for every scenario, ``saa_mean`` finalizes the SAA statistics,
``irp_dp`` runs the inventory-routing recourse DP (DESIGN R21).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspdp.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        "paper_2511_18022_b200: %s is missing -- build it with "
        "`python -m paper_2511_18022_b200.build` (nvcc, sm_100a). There is no CPU fallback." % LIB_PATH)

_lib = ctypes.CDLL(LIB_PATH)

SPDP_OK, SPDP_E_USAGE, SPDP_E_DATA, SPDP_E_RESOURCE, SPDP_E_CUDA = 0, 2, 3, 4, 5
INFEASIBLE = 2**31 - 1
F_VALIDATE = 1
F_SCRATCH_GLOBAL = 16
F_NBR_SMEM = 32
F_NBR_AUTO = 64
F_SWEEP = {None: 0, "auto": 0, "int": 2, "f32": 4, "deque": 8, "u16": 128}
F_IRP_EAGER = 65536  # sweep algorithm flags (spdp.h)
F_IRP_STATES = 131072
MAX_N = 16384

SYMBOLS = (
    "spdp_version", "spdp_last_error", "spdp_workspace_bytes", "spdp_gen_demands", "spdp_demand_prefix",
    "spdp_split_mask", "spdp_split_eval", "spdp_split_eval_batch", "spdp_saa_reduce", "spdp_saa_mean",
    "spdp_host_workspace_bytes", "spdp_split_eval_host", "spdp_irp_workspace_bytes", "spdp_irp_dp",
    "spdp_set_profile_events", "spdp_last_kernel", "spdp_debug_timeline", "spdp_routes_workspace_bytes", "spdp_split_routes",
    "spdp_split_eval_penalized", "spdp_values_workspace_bytes", "spdp_split_values",
    "spdp_neighbour_workspace_bytes", "spdp_split_eval_neighbours", "spdp_limits_workspace_bytes",
    "spdp_split_eval_limits", "spdp_f32_workspace_bytes", "spdp_split_eval_f32", "spdp_saa_estimate_f32",
    "spdp_saa_f32_moments", "spdp_saa_finalize_f32", "spdp_split_eval_batch_f32", "spdp_split_eval_neighbours_multi",
    "spdp_order_workspace_bytes", "spdp_order_scenarios",
)


class SaaPartial(ctypes.Structure):
    _fields_ = [("n_feas", ctypes.c_int64), ("n_infeas", ctypes.c_int64), ("sum", ctypes.c_int64),
                ("sumsq_lo", ctypes.c_int64), ("sumsq_hi", ctypes.c_int64), ("reserved", ctypes.c_int64)]


class SaaEstimate(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int64), ("infeasible", ctypes.c_int64), ("mean", ctypes.c_double),
                ("var", ctypes.c_double), ("std_err", ctypes.c_double), ("ci95_lo", ctypes.c_double),
                ("ci95_hi", ctypes.c_double)]


class DemandModel(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("n", ctypes.c_int32), ("nominal", ctypes.c_void_p),
                ("lo_pm", ctypes.c_int32), ("hi_pm", ctypes.c_int32), ("A_fx", ctypes.c_int64),
                ("B_fx", ctypes.c_int64), ("q_cap", ctypes.c_int32), ("stream_tag", ctypes.c_uint32),
                ("seed", ctypes.c_uint64)]


class IrpCustomer(ctypes.Structure):
    _fields_ = [("U", ctypes.c_int32), ("X", ctypes.c_int32), ("I0", ctypes.c_int32), ("h", ctypes.c_int32),
                ("b", ctypes.c_int32), ("c", ctypes.c_int32)]


def _sig():
    P, i32, i64, u32, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_size_t
    st = ctypes.c_int
    L = _lib
    L.spdp_version.restype = ctypes.c_int
    L.spdp_set_profile_events.argtypes = [P, P]
    L.spdp_set_profile_events.restype = None
    L.spdp_last_error.restype = ctypes.c_char_p
    L.spdp_last_kernel.restype = ctypes.c_char_p
    L.spdp_debug_timeline.argtypes = [ctypes.c_void_p]
    L.spdp_debug_timeline.restype = ctypes.c_int
    L.spdp_workspace_bytes.argtypes = [i32, i64, i32]
    L.spdp_workspace_bytes.restype = sz
    L.spdp_host_workspace_bytes.argtypes = [i32, i64]
    L.spdp_host_workspace_bytes.restype = sz
    L.spdp_irp_workspace_bytes.argtypes = [i32, i32, i64]
    L.spdp_irp_workspace_bytes.restype = sz
    L.spdp_gen_demands.argtypes = [ctypes.POINTER(DemandModel), i64, i64, P, i64, P]
    L.spdp_demand_prefix.argtypes = [P, i32, P, i64, i64, P, P]
    L.spdp_split_mask.argtypes = [P, i32, P, i64, i64, i32, P, P]
    L.spdp_split_eval.argtypes = [P, P, i32, P, i64, i64, i32, P, P, i32, P, sz, u32, P]
    L.spdp_split_eval_batch.argtypes = [P, i32, P, i32, P, i64, i64, i32, P, P, i32, P, sz, u32, P]
    L.spdp_saa_reduce.argtypes = [P, i64, P, P]
    L.spdp_split_eval_penalized.argtypes = [P, P, i32, P, i64, i64, i32, i32, P, P, i32, P, sz, u32, P]
    L.spdp_routes_workspace_bytes.argtypes = [i32, i32]
    L.spdp_routes_workspace_bytes.restype = sz
    L.spdp_split_routes.argtypes = [P, P, i32, P, i64, i64, i32, P, i32, P, P, P, P, P, sz, P]
    L.spdp_values_workspace_bytes.argtypes = [i32, i64]
    L.spdp_values_workspace_bytes.restype = sz
    L.spdp_split_values.argtypes = [P, P, i32, P, i64, i64, i32, P, P, P, sz, P]
    L.spdp_neighbour_workspace_bytes.argtypes = [i32, i64, i32]
    L.spdp_neighbour_workspace_bytes.restype = sz
    L.spdp_split_eval_neighbours.argtypes = [P, P, P, P, i32, P, i32, P, i64, i64, i32, P, P, i32, P, sz, u32, P]
    L.spdp_split_eval_neighbours_multi.argtypes = [P, i32, P, P, P, P, i32, P, i32, P, i64, i64, i32, P, P, i32, P, sz,
                                                   u32, P]
    L.spdp_limits_workspace_bytes.argtypes = [i32, i64]
    L.spdp_limits_workspace_bytes.restype = sz
    L.spdp_split_eval_limits.argtypes = [P, P, i32, P, i64, i64, i32, i32, i32, P, P, P, sz, u32, P]
    L.spdp_f32_workspace_bytes.argtypes = [i32, i64]
    L.spdp_f32_workspace_bytes.restype = sz
    L.spdp_split_eval_f32.argtypes = [P, P, i32, P, i64, i64, i32, P, P, sz, P]
    L.spdp_saa_estimate_f32.argtypes = [P, i64, ctypes.POINTER(SaaEstimate), P, sz, P]
    L.spdp_saa_f32_moments.argtypes = [P, i64, ctypes.c_double, P, P]
    L.spdp_saa_finalize_f32.argtypes = [P, P, ctypes.POINTER(SaaEstimate)]
    L.spdp_split_eval_batch_f32.argtypes = [P, i32, P, i32, P, i64, i64, i32, P, P, sz, P]
    L.spdp_saa_mean.argtypes = [ctypes.POINTER(SaaPartial), ctypes.POINTER(SaaEstimate)]
    L.spdp_order_workspace_bytes.argtypes = [i64]
    L.spdp_order_workspace_bytes.restype = sz
    L.spdp_order_scenarios.argtypes = [P, i64, i32, i64, P, i64, P, P, sz, P]
    L.spdp_split_eval_host.argtypes = [P, P, i32, P, i64, i64, i32, P, ctypes.POINTER(SaaEstimate), i32, P, sz, P]
    L.spdp_irp_dp.argtypes = [P, ctypes.POINTER(IrpCustomer), i32, i32, P, i64, i64, P, P, P, sz, u32, P]
    for name in ("spdp_gen_demands", "spdp_demand_prefix", "spdp_split_mask", "spdp_split_eval",
                 "spdp_split_eval_batch", "spdp_saa_reduce", "spdp_saa_mean", "spdp_split_eval_host",
                 "spdp_irp_dp", "spdp_split_values", "spdp_split_eval_neighbours", "spdp_split_eval_penalized",
                 "spdp_split_routes", "spdp_split_eval_limits", "spdp_split_eval_f32", "spdp_saa_estimate_f32",
                 "spdp_saa_f32_moments", "spdp_saa_finalize_f32", "spdp_split_eval_batch_f32",
                 "spdp_split_eval_neighbours_multi", "spdp_order_scenarios"):
        getattr(L, name).restype = st


_sig()


class SpdpError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = _lib.spdp_last_error().decode(errors="replace")
        super().__init__("%s failed (status %d): %s" % (where, status, msg))
        self.status = status


def _check(rc: int, where: str):
    if rc != SPDP_OK:
        raise SpdpError(rc, where)


def set_profile_events(start=None, stop=None):
    """Record torch.cuda.Event pair (start, stop) around the dominant kernel of the next calls
    on this thread (the sweep / IRP kernel); call with no arguments to clear.  The events must
    already exist (torch creates them lazily: record them once first)."""
    if start is None or stop is None:
        _lib.spdp_set_profile_events(None, None)
    else:
        if not start.cuda_event or not stop.cuda_event:
            raise ValueError("set_profile_events: events not created yet (record them once first)")
        _lib.spdp_set_profile_events(ctypes.c_void_p(start.cuda_event), ctypes.c_void_p(stop.cuda_event))


def last_kernel() -> str:
    """Name of the sweep kernel the last split call on this thread enqueued (spdp_last_kernel)."""
    return _lib.spdp_last_kernel().decode()


def debug_timeline(buf=None):
    """Debug timeline of the u16 sweep (spdp_debug_timeline): a zeroed int64 CUDA tensor receives
    per-tile records from later sweeps; None switches it off.  Measurement only."""
    _check(_lib.spdp_debug_timeline(ctypes.c_void_p(0 if buf is None else buf.data_ptr())), "spdp_debug_timeline")


def version() -> int:
    return int(_lib.spdp_version())


def lib():
    """The raw ctypes handle of libspdp.so."""
    return _lib


# ------------------------------------------------------------------ torch plumbing
def _torch():
    import torch
    return torch


def _dev_ptr(t, what: str):
    torch = _torch()
    if t is None:
        return None
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError("%s must be a CUDA tensor (the kernels have no CPU path)" % what)
    if not t.is_contiguous():
        raise ValueError("%s must be contiguous" % what)
    return ctypes.c_void_p(t.data_ptr())


def _stream(device):
    torch = _torch()
    return ctypes.c_void_p(torch.cuda.current_stream(device).cuda_stream)


_WS = {}


def _mean_flag(mean_window: int) -> int:
    """flags bits 8..15: expected mean window (spdp.h SPDP_F_MEAN_WINDOW)."""
    return (min(max(int(mean_window), 0), 255)) << 8


def workspace(nbytes: int, device, tag: str = "split"):
    """Cached scratch buffer (torch uint8) per (device, current stream, tag), grown on demand.

    spdp.h forbids one workspace in two concurrent calls: keying by the stream gives calls on
    different streams (or threads using different streams) their own buffers.  A grown buffer's
    predecessor is released only after the stream has finished with it (record_stream), and a
    captured CUDA graph keeps referring to the buffer it was captured with -- replay it only while
    that buffer is alive (a graph pins its workspace; bench.py holds a reference)."""
    torch = _torch()
    dev = torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    stream = torch.cuda.current_stream(idx)
    key = (idx, stream.cuda_stream, tag)
    buf = _WS.get(key)
    if buf is None or buf.numel() < nbytes:
        if buf is not None:
            buf.record_stream(stream)  # the caching allocator reuses it only after the stream's queued work
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=dev)
        _WS[key] = buf
    return buf


def _default_S(demand, S):
    """The scenario count of a demand matrix: S if given, else the true count recorded by
    gen_demands / empty_demand (not the padded row length ld, whose padding columns would be
    evaluated as extra all-zero scenarios), else ld."""
    if S is not None:
        return int(S)
    return int(getattr(demand, "_spdp_S", demand.shape[1]))


def workspace_bytes(n: int, S: int, T: int = 1) -> int:
    return int(_lib.spdp_workspace_bytes(n, S, T))


def padded_ld(S: int) -> int:
    return (S + 7) // 8 * 8


def empty_demand(n: int, S: int, device):
    """u16 demand matrix [n][ld] (stored as torch.int16), ld = S rounded up to 8; the true S is
    recorded on the tensor (the default S of every call that takes it)."""
    torch = _torch()
    out = torch.zeros((n, padded_ld(S)), dtype=torch.int16, device=device)
    out._spdp_S = int(S)
    return out


# ------------------------------------------------------------------ a1
def gen_demands(model: dict, s_begin: int, S: int, device="cuda", out=None):
    """Generate the demand shard [n][ld] for global scenarios [s_begin, s_begin+S)."""
    torch = _torch()
    nominal = torch.as_tensor(np.ascontiguousarray(model["nominal"], dtype=np.uint16).view(np.int16),
                              device=device)
    n = nominal.shape[0]
    if out is None:
        out = empty_demand(n, S, device)
    m = DemandModel(kind=int(model["kind"]), n=n, nominal=nominal.data_ptr(), lo_pm=int(model.get("lo_pm", 0)),
                    hi_pm=int(model.get("hi_pm", 0)), A_fx=int(model.get("A_fx", 0)), B_fx=int(model.get("B_fx", 0)),
                    q_cap=int(model["q_cap"]), stream_tag=int(model.get("stream_tag", 0)), seed=int(model["seed"]))
    _check(_lib.spdp_gen_demands(ctypes.byref(m), int(s_begin), int(S), _dev_ptr(out, "out"), out.shape[1],
                                 _stream(out.device)), "spdp_gen_demands")
    out._spdp_S = int(S)
    out._spdp_nominal = nominal  # keep alive until the stream has consumed it
    return out


def order_scenarios(demand, S: int | None = None, out=None, want_out: bool = True):
    """a1 layout: the scenarios (columns) of `demand` in increasing bucketed total demand
    (spdp_order_scenarios).  Returns (ordered demand [n][ld] or None, perm int32 [S]):
    column j of the result is scenario perm[j] of `demand`."""
    torch = _torch()
    n, ld = demand.shape
    S = _default_S(demand, S)
    perm = torch.empty(S, dtype=torch.int32, device=demand.device)
    if want_out and out is None:
        out = empty_demand(n, S, demand.device)
    ws = workspace(int(_lib.spdp_order_workspace_bytes(S)), demand.device, tag="order")
    _check(_lib.spdp_order_scenarios(_dev_ptr(demand, "demand"), ld, n, S, _dev_ptr(out, "out") if want_out else None,
                                     out.shape[1] if want_out else 0, _dev_ptr(perm, "perm"), _dev_ptr(ws, "ws"),
                                     ws.numel(), _stream(demand.device)), "spdp_order_scenarios")
    if want_out:
        out._spdp_S = int(S)
    return (out if want_out else None), perm


# ------------------------------------------------------------------ a3 / a4
def demand_prefix(tour, demand, S: int | None = None):
    torch = _torch()
    n, ld = demand.shape
    S = _default_S(demand, S)
    out = torch.empty((n + 1, S), dtype=torch.int32, device=demand.device)
    _check(_lib.spdp_demand_prefix(_dev_ptr(tour, "tour"), n, _dev_ptr(demand, "demand"), ld, S,
                                   _dev_ptr(out, "prefix"), _stream(demand.device)), "spdp_demand_prefix")
    return out


def split_mask(tour, demand, Q: int, S: int | None = None):
    torch = _torch()
    n, ld = demand.shape
    S = _default_S(demand, S)
    out = torch.empty((n, S), dtype=torch.int32, device=demand.device)
    _check(_lib.spdp_split_mask(_dev_ptr(tour, "tour"), n, _dev_ptr(demand, "demand"), ld, S, int(Q),
                                _dev_ptr(out, "mask"), _stream(demand.device)), "spdp_split_mask")
    return out


# ------------------------------------------------------------------ a2 + a5 + a6
def split_eval(tour, dist, demand, Q: int, S: int | None = None, want_cost: bool = True,
               want_partial: bool = True, window_hint: int = 0, validate: bool = False, cost=None, partial=None,
               algo: str | None = None, mean_window: int = 0):
    """Per-scenario split costs (int32 [S], INFEASIBLE sentinel) and the SAA partial (int64 [6]).
    algo: None/"auto", "int", "f32", "deque" or "u16" (identical results; see spdp.h)."""
    torch = _torch()
    n, ld = demand.shape
    S = _default_S(demand, S)
    dev = demand.device
    if want_cost and cost is None:
        cost = torch.empty(S, dtype=torch.int32, device=dev)
    if want_partial and partial is None:
        partial = torch.zeros(6, dtype=torch.int64, device=dev)
    nb = workspace_bytes(n, S, 1)
    ws = workspace(nb, dev)
    _check(_lib.spdp_split_eval(_dev_ptr(tour, "tour"), _dev_ptr(dist, "dist"), n, _dev_ptr(demand, "demand"), ld, S,
                                int(Q), _dev_ptr(cost, "cost") if want_cost else None,
                                _dev_ptr(partial, "partial") if want_partial else None, int(window_hint),
                                ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                (F_VALIDATE if validate else 0) | F_SWEEP[algo] | _mean_flag(mean_window),
                                _stream(dev)), "spdp_split_eval")
    return cost, partial


def split_eval_penalized(tour, dist, demand, Q: int, lam: int, S: int | None = None, want_cost: bool = True,
                         want_partial: bool = True, window_hint: int = 0, validate: bool = False, cost=None,
                         partial=None):
    """f2: penalized split costs (int32 [S]) and the SAA partial (spdp_split_eval_penalized)."""
    torch = _torch()
    n, ld = demand.shape
    S = _default_S(demand, S)
    dev = demand.device
    if want_cost and cost is None:
        cost = torch.empty(S, dtype=torch.int32, device=dev)
    if want_partial and partial is None:
        partial = torch.zeros(6, dtype=torch.int64, device=dev)
    ws = workspace(workspace_bytes(n, S, 1), dev)
    _check(_lib.spdp_split_eval_penalized(_dev_ptr(tour, "tour"), _dev_ptr(dist, "dist"), n, _dev_ptr(demand, "demand"),
                                          ld, S, int(Q), int(lam), _dev_ptr(cost, "cost") if want_cost else None,
                                          _dev_ptr(partial, "partial") if want_partial else None, int(window_hint),
                                          ctypes.c_void_p(ws.data_ptr()), ws.numel(), F_VALIDATE if validate else 0,
                                          _stream(dev)), "spdp_split_eval_penalized")
    return cost, partial


def split_routes(tour, dist, demand, Q: int, scen, S: int | None = None):
    """f1: optimal routes of K selected scenarios (spdp_split_routes).
    scen: int64 tensor [K] of scenario indices.  Returns (cost int32 [K], pred int32 [K][n+1],
    nroutes int32 [K], maxload int32 [K]); pred[k][i] = last split point of prefix i."""
    torch = _torch()
    n, ld = demand.shape
    S = _default_S(demand, S)
    dev = demand.device
    K = int(scen.shape[0])
    cost = torch.empty(K, dtype=torch.int32, device=dev)
    pred = torch.empty((K, n + 1), dtype=torch.int32, device=dev)
    nroutes = torch.empty(K, dtype=torch.int32, device=dev)
    maxload = torch.empty(K, dtype=torch.int32, device=dev)
    nb = int(_lib.spdp_routes_workspace_bytes(n, K))
    ws = workspace(nb, dev, tag="routes")
    _check(_lib.spdp_split_routes(_dev_ptr(tour, "tour"), _dev_ptr(dist, "dist"), n, _dev_ptr(demand, "demand"), ld, S,
                                  int(Q), _dev_ptr(scen, "scen"), K, _dev_ptr(pred, "pred"), _dev_ptr(cost, "cost"),
                                  _dev_ptr(nroutes, "nroutes"), _dev_ptr(maxload, "maxload"),
                                  ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream(dev)), "spdp_split_routes")
    return cost, pred, nroutes, maxload


def split_eval_batch(tours, dist, demand, Q: int, S: int | None = None, want_cost: bool = True,
                     want_partial: bool = True, window_hint: int = 0, validate: bool = False, cost=None,
                     partial=None, algo: str | None = None, mean_window: int = 0):
    """T tours [T][n] over one demand set: costs int32 [T][S] and partials int64 [T][6]."""
    torch = _torch()
    n, ld = demand.shape
    T = tours.shape[0]
    S = _default_S(demand, S)
    dev = demand.device
    if want_cost and cost is None:
        cost = torch.empty((T, S), dtype=torch.int32, device=dev)
    if want_partial and partial is None:
        partial = torch.zeros((T, 6), dtype=torch.int64, device=dev)
    ws = workspace(workspace_bytes(n, S, T), dev)
    _check(_lib.spdp_split_eval_batch(_dev_ptr(tours, "tours"), T, _dev_ptr(dist, "dist"), n,
                                      _dev_ptr(demand, "demand"), ld, S, int(Q),
                                      _dev_ptr(cost, "cost") if want_cost else None,
                                      _dev_ptr(partial, "partial") if want_partial else None, int(window_hint),
                                      ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                      (F_VALIDATE if validate else 0) | F_SWEEP[algo] | _mean_flag(mean_window), _stream(dev)),
           "spdp_split_eval_batch")
    return cost, partial


def split_values(tour, dist, demand, Q: int, S: int | None = None, fwd=None, bwd=None):
    """f3: prefix / suffix split values of one tour (spdp_split_values).
    Returns (fwd, bwd), int32 [n+1][S] each: fwd[i] = Split of the first i customers,
    bwd[i] = Split of the customers after position i (INFEASIBLE sentinel)."""
    torch = _torch()
    n, ld = demand.shape
    S = _default_S(demand, S)
    dev = demand.device
    if fwd is None:
        fwd = torch.empty((n + 1, S), dtype=torch.int32, device=dev)
    if bwd is None:
        bwd = torch.empty((n + 1, S), dtype=torch.int32, device=dev)
    ws = workspace(int(_lib.spdp_values_workspace_bytes(n, S)), dev, tag="values")
    _check(_lib.spdp_split_values(_dev_ptr(tour, "tour"), _dev_ptr(dist, "dist"), n, _dev_ptr(demand, "demand"), ld, S,
                                  int(Q), _dev_ptr(fwd, "fwd"), _dev_ptr(bwd, "bwd"), ctypes.c_void_p(ws.data_ptr()),
                                  ws.numel(), _stream(dev)), "spdp_split_values")
    return fwd, bwd


def split_eval_neighbours(parent, fwd, bwd, tours, dist, demand, Q: int, S: int | None = None,
                          want_cost: bool = True, want_partial: bool = True, window_hint: int = 0,
                          validate: bool = False, cost=None, partial=None, smem: bool = False,
                          int_only: bool = False, auto: bool = False, mean_window: int = 0):
    """f3: split costs of T candidate tours [T][n] from the parent's values (spdp_split_eval_neighbours);
    bit-identical to split_eval_batch(tours, ...).  Returns (cost int32 [T][S], partial int64 [T][6]).
    smem: the shared-memory-ring kernel instead of the register ring; int_only: no exact-fp32 phase
    (SPDP_F_SWEEP_INT); auto: the batched sweep when the changed spans are long (SPDP_F_NBR_AUTO,
    synchronizes; mean_window is then its tuning hint as in split_eval_batch); same results in every case."""
    torch = _torch()
    n, ld = demand.shape
    T = tours.shape[0]
    S = _default_S(demand, S)
    dev = demand.device
    if want_cost and cost is None:
        cost = torch.empty((T, S), dtype=torch.int32, device=dev)
    if want_partial and partial is None:
        partial = torch.zeros((T, 6), dtype=torch.int64, device=dev)
    ws = workspace(int(_lib.spdp_neighbour_workspace_bytes(n, S, T)), dev, tag="nbr")
    _check(_lib.spdp_split_eval_neighbours(_dev_ptr(parent, "parent"), _dev_ptr(fwd, "fwd"), _dev_ptr(bwd, "bwd"),
                                           _dev_ptr(tours, "tours"), T, _dev_ptr(dist, "dist"), n,
                                           _dev_ptr(demand, "demand"), ld, S, int(Q),
                                           _dev_ptr(cost, "cost") if want_cost else None,
                                           _dev_ptr(partial, "partial") if want_partial else None, int(window_hint),
                                           ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                           (F_VALIDATE if validate else 0) | (F_NBR_SMEM if smem else 0) | (F_SWEEP["int"] if int_only else 0)
                                           | (F_NBR_AUTO if auto else 0) | _mean_flag(mean_window),
                                           _stream(dev)),
           "spdp_split_eval_neighbours")
    return cost, partial


def split_eval_limits(tour, dist, demand, Q: int, max_duration: int = -1, max_routes: int = 0,
                      S: int | None = None, want_cost: bool = True, want_partial: bool = True, cost=None,
                      partial=None, scratch_global: bool = False):
    """f4: split costs with a route-duration limit (route cost <= max_duration; < 0: none) and at
    most max_routes routes (<= 0: none) (spdp_split_eval_limits).  Returns (cost int32 [S], partial)."""
    torch = _torch()
    n, ld = demand.shape
    S = _default_S(demand, S)
    dev = demand.device
    if want_cost and cost is None:
        cost = torch.empty(S, dtype=torch.int32, device=dev)
    if want_partial and partial is None:
        partial = torch.zeros(6, dtype=torch.int64, device=dev)
    ws = workspace(int(_lib.spdp_limits_workspace_bytes(n, S)), dev, tag="limits")
    _check(_lib.spdp_split_eval_limits(_dev_ptr(tour, "tour"), _dev_ptr(dist, "dist"), n, _dev_ptr(demand, "demand"),
                                       ld, S, int(Q), int(max_duration), int(max_routes),
                                       _dev_ptr(cost, "cost") if want_cost else None,
                                       _dev_ptr(partial, "partial") if want_partial else None,
                                       ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                       F_SCRATCH_GLOBAL if scratch_global else 0, _stream(dev)),
           "spdp_split_eval_limits")
    return cost, partial


def split_eval_f32(tour, dist, demand, Q: int, S: int | None = None, cost=None):
    """a5 fp32 mode (spdp_split_eval_f32): dist a CUDA float64 tensor [(n+1)^2] of real costs;
    returns float32 costs [S] (+inf = infeasible)."""
    torch = _torch()
    n, ld = demand.shape
    S = _default_S(demand, S)
    dev = demand.device
    if cost is None:
        cost = torch.empty(S, dtype=torch.float32, device=dev)
    ws = workspace(int(_lib.spdp_f32_workspace_bytes(n, S)), dev, tag="f32")
    _check(_lib.spdp_split_eval_f32(_dev_ptr(tour, "tour"), _dev_ptr(dist, "dist"), n, _dev_ptr(demand, "demand"), ld,
                                    S, int(Q), _dev_ptr(cost, "cost"), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                    _stream(dev)), "spdp_split_eval_f32")
    return cost


def split_eval_batch_f32(tours, dist, demand, Q: int, S: int | None = None, cost=None):
    """a8 in fp32 mode (spdp_split_eval_batch_f32): float32 costs [T][S] of T tours [T][n]."""
    torch = _torch()
    n, ld = demand.shape
    T = tours.shape[0]
    S = _default_S(demand, S)
    dev = demand.device
    if cost is None:
        cost = torch.empty((T, S), dtype=torch.float32, device=dev)
    ws = workspace(int(_lib.spdp_f32_workspace_bytes(n, S)), dev, tag="f32")
    _check(_lib.spdp_split_eval_batch_f32(_dev_ptr(tours, "tours"), T, _dev_ptr(dist, "dist"), n,
                                          _dev_ptr(demand, "demand"), ld, S, int(Q), _dev_ptr(cost, "cost"),
                                          ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream(dev)),
           "spdp_split_eval_batch_f32")
    return cost


def saa_estimate_f32(cost) -> dict:
    """SAA estimate of float32 costs on the device (spdp_saa_estimate_f32; synchronizes)."""
    ws = workspace(64, cost.device, tag="saa_f32")
    e = SaaEstimate()
    _check(_lib.spdp_saa_estimate_f32(_dev_ptr(cost, "cost"), cost.numel(), ctypes.byref(e),
                                      ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream(cost.device)),
           "spdp_saa_estimate_f32")
    return {"m": e.m, "infeasible": e.infeasible, "mean": e.mean, "var": e.var, "stderr": e.std_err,
            "ci95_lo": e.ci95_lo, "ci95_hi": e.ci95_hi}


def saa_f32_moments(cost, center: float = 0.0, out=None):
    """{m, sum, sum (c - center)^2, infeasible} of float32 costs (DEVICE float64 [4], asynchronous)."""
    torch = _torch()
    if out is None:
        out = torch.empty(4, dtype=torch.float64, device=cost.device)
    _check(_lib.spdp_saa_f32_moments(_dev_ptr(cost, "cost"), cost.numel(), float(center), _dev_ptr(out, "moments"),
                                     _stream(cost.device)), "spdp_saa_f32_moments")
    return out


def saa_finalize_f32(m1, m2=None) -> dict:
    """fp32-mode SAA estimate (spdp_saa_finalize_f32, host) from summed pass-1 moments m1 and,
    optionally, the pass-2 moments m2 centred on the pass-1 mean (float64 [4] each, any device)."""
    a1 = np.ascontiguousarray(m1.detach().cpu().numpy() if hasattr(m1, "detach") else m1, dtype=np.float64).reshape(4)
    a2 = None
    if m2 is not None:
        a2 = np.ascontiguousarray(m2.detach().cpu().numpy() if hasattr(m2, "detach") else m2,
                                  dtype=np.float64).reshape(4)
    e = SaaEstimate()
    _check(_lib.spdp_saa_finalize_f32(a1.ctypes.data_as(ctypes.c_void_p),
                                      a2.ctypes.data_as(ctypes.c_void_p) if a2 is not None else None,
                                      ctypes.byref(e)), "spdp_saa_finalize_f32")
    return {"m": e.m, "infeasible": e.infeasible, "mean": e.mean, "var": e.var, "stderr": e.std_err,
            "ci95_lo": e.ci95_lo, "ci95_hi": e.ci95_hi}


def split_eval_neighbours_multi(parents, parent_of, fwd, bwd, tours, dist, demand, Q: int, S: int | None = None,
                                want_cost: bool = True, want_partial: bool = True, window_hint: int = 0,
                                cost=None, partial=None):
    """f3 with several parents (spdp_split_eval_neighbours_multi): parents int32 [P][n], parent_of int32 [T],
    fwd / bwd int32 [P][n+1][S] (stacked split_values of each parent)."""
    torch = _torch()
    n, ld = demand.shape
    T = tours.shape[0]
    P = parents.shape[0]
    S = _default_S(demand, S)
    dev = demand.device
    if want_cost and cost is None:
        cost = torch.empty((T, S), dtype=torch.int32, device=dev)
    if want_partial and partial is None:
        partial = torch.zeros((T, 6), dtype=torch.int64, device=dev)
    ws = workspace(int(_lib.spdp_neighbour_workspace_bytes(n, S, T)), dev, tag="nbr")
    _check(_lib.spdp_split_eval_neighbours_multi(_dev_ptr(parents, "parents"), P, _dev_ptr(parent_of, "parent_of"),
                                                 _dev_ptr(fwd, "fwd"), _dev_ptr(bwd, "bwd"), _dev_ptr(tours, "tours"), T,
                                                 _dev_ptr(dist, "dist"), n, _dev_ptr(demand, "demand"), ld, S, int(Q),
                                                 _dev_ptr(cost, "cost") if want_cost else None,
                                                 _dev_ptr(partial, "partial") if want_partial else None,
                                                 int(window_hint), ctypes.c_void_p(ws.data_ptr()), ws.numel(), 0,
                                                 _stream(dev)), "spdp_split_eval_neighbours_multi")
    return cost, partial


def saa_reduce(cost, partial=None):
    torch = _torch()
    if partial is None:
        partial = torch.zeros(6, dtype=torch.int64, device=cost.device)
    _check(_lib.spdp_saa_reduce(_dev_ptr(cost, "cost"), cost.numel(), _dev_ptr(partial, "partial"),
                                _stream(cost.device)), "spdp_saa_reduce")
    return partial


def saa_mean(partial) -> dict:
    """Host finalize of an SAA partial (int64[6] tensor/array, any device)."""
    arr = partial.detach().cpu().numpy() if hasattr(partial, "detach") else np.asarray(partial)
    arr = np.ascontiguousarray(arr, dtype=np.int64).reshape(6)
    p = SaaPartial(*[int(v) for v in arr])
    e = SaaEstimate()
    _check(_lib.spdp_saa_mean(ctypes.byref(p), ctypes.byref(e)), "spdp_saa_mean")
    return {"m": e.m, "infeasible": e.infeasible, "mean": e.mean, "var": e.var, "stderr": e.std_err,
            "ci95_lo": e.ci95_lo, "ci95_hi": e.ci95_hi}


def host_workspace_bytes(n: int, S: int) -> int:
    return int(_lib.spdp_host_workspace_bytes(n, S))


def split_eval_host(tour_h, dist_h, demand_h, Q: int, S: int | None = None, cost_h=None, window_hint: int = 0,
                    device="cuda"):
    """End-to-end call with HOST buffers (numpy or pinned torch CPU tensors): H2D copy, kernels,
    D2H of the estimate (and of cost_h if given).  Returns the SAA estimate dict."""
    torch = _torch()

    def hptr(a, what):
        if a is None:
            return None
        if isinstance(a, torch.Tensor):
            if a.is_cuda or not a.is_contiguous():
                raise ValueError("%s must be a contiguous CPU tensor" % what)
            return ctypes.c_void_p(a.data_ptr())
        a = np.asarray(a)
        if not a.flags["C_CONTIGUOUS"]:
            raise ValueError("%s must be C-contiguous" % what)
        return a.ctypes.data_as(ctypes.c_void_p)

    n, ld = demand_h.shape
    S = _default_S(demand_h, S)
    ws = workspace(host_workspace_bytes(n, S), device, tag="host")
    e = SaaEstimate()
    _check(_lib.spdp_split_eval_host(hptr(tour_h, "tour"), hptr(dist_h, "dist"), n, hptr(demand_h, "demand"), ld, S,
                                     int(Q), hptr(cost_h, "cost"), ctypes.byref(e), int(window_hint),
                                     ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream(torch.device(device))),
           "spdp_split_eval_host")
    return {"m": e.m, "infeasible": e.infeasible, "mean": e.mean, "var": e.var, "stderr": e.std_err,
            "ci95_lo": e.ci95_lo, "ci95_hi": e.ci95_hi}


# ------------------------------------------------------------------ a9 + a10
def irp_dp(visit, cust, demand, H: int, M: int, S: int | None = None, want_partial: bool = True, cost=None,
           partial=None, eager: bool = False, states: bool = False):
    """IRP recourse cost per scenario (int64 [S]); visit u8 [M][H] and cust int32 [M][6] on the host.
    eager: the eager-shift kernel (SPDP_F_IRP_EAGER); states: the state-parallel kernel
    (SPDP_F_IRP_STATES); same results."""
    torch = _torch()
    ld = demand.shape[1]
    S = _default_S(demand, S)
    dev = demand.device
    visit = np.ascontiguousarray(visit, dtype=np.uint8)
    cust = np.ascontiguousarray(cust, dtype=np.int32)
    carr = (IrpCustomer * M)(*[IrpCustomer(*[int(v) for v in row]) for row in cust])
    if cost is None:
        cost = torch.empty(S, dtype=torch.int64, device=dev)
    if want_partial and partial is None:
        partial = torch.zeros(6, dtype=torch.int64, device=dev)
    ws = workspace(int(_lib.spdp_irp_workspace_bytes(H, M, S)), dev, tag="irp")
    _check(_lib.spdp_irp_dp(visit.ctypes.data_as(ctypes.c_void_p), carr, H, M, _dev_ptr(demand, "demand"), ld, S,
                            _dev_ptr(cost, "cost"), _dev_ptr(partial, "partial") if want_partial else None,
                            ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                            (F_IRP_EAGER if eager else 0) | (F_IRP_STATES if states else 0), _stream(dev)),
           "spdp_irp_dp")
    return cost, partial
