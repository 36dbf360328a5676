"""ctypes binding of libkfac.so (include/kfac.h) -- argument marshalling only.

Every function here has the name of the C entry point it wraps (without the
``kfac_`` prefix) and forwards device pointers of torch CUDA tensors plus the
current CUDA stream; all computation happens in the library's kernels / NCCL.
There is no fallback: if libkfac.so is missing, importing this module fails.
"""
from __future__ import annotations

import ctypes
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libkfac.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with `python -m paper_1811_12019_b200.build` "
                      "(there is no CPU fallback for the K-FAC hot path)")

_lib = ctypes.CDLL(LIB_PATH)

BF16, FP16 = 0, 1
RR, LPT = 0, 1
_DT = {torch.bfloat16: BF16, torch.float16: FP16}

STATUS = {0: "OK", 1: "ERR_ARG", 2: "ERR_SHAPE", 3: "ERR_UNSUPPORTED", 4: "ERR_CUDA", 5: "ERR_NCCL",
          6: "ERR_NOT_PD", 7: "ERR_STATE"}


class KfacError(RuntimeError):
    def __init__(self, status, where):
        self.status = status
        msg = _lib.kfac_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg}")


class LayerDesc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("kind", "c_in", "c_out", "kh", "kw", "stride_h", "stride_w", "pad_h", "pad_w", "h_in", "w_in",
                 "has_bias")]


def layer_desc(d: dict) -> LayerDesc:
    return LayerDesc(*(int(d[k]) for k, _ in LayerDesc._fields_))


_P = ctypes.c_void_p
_i32, _i64, _f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float
_pi32, _pi64 = ctypes.POINTER(ctypes.c_int32), ctypes.POINTER(ctypes.c_int64)
_pf32 = ctypes.POINTER(ctypes.c_float)


def _sig(name, args):
    f = getattr(_lib, name)
    f.argtypes = args
    f.restype = ctypes.c_int
    return f


_lib.kfac_last_error.restype = ctypes.c_char_p
_lib.kfac_version.restype = ctypes.c_char_p
_lib.kfac_launch_count.restype = ctypes.c_int64
_lib.kfac_launch_count.argtypes = []
_lib.kfac_plan_destroy.argtypes = [_P]
_lib.kfac_plan_destroy.restype = None
_lib.kfac_comm_destroy.argtypes = [_P]
_lib.kfac_comm_destroy.restype = None
_plan_create = _sig("kfac_plan_create", [ctypes.POINTER(LayerDesc), _i32, _i32, _i32, ctypes.c_int, ctypes.POINTER(_P)])
_plan_query = _sig("kfac_plan_query", [_P, _pi32, _pi64, _pi64, _pi64, _pi64, _pi64])
_plan_rank_layers = _sig("kfac_plan_rank_layers", [_P, _i32, _pi32, _pi32, _pi64, _pi64, _pi64])
_comm_unique_id = _sig("kfac_comm_unique_id", [ctypes.c_char_p])
_comm_create = _sig("kfac_comm_create", [ctypes.c_char_p, _i32, _i32, _i32, ctypes.POINTER(_P)])
_factor_A = _sig("kfac_factor_A", [ctypes.POINTER(LayerDesc), _P, ctypes.c_int, _i32, _f32, _P, _P, _i64, _P])
_factor_G = _sig("kfac_factor_G", [ctypes.POINTER(LayerDesc), _P, ctypes.c_int, _i32, _f32, _P, _P, _i64, _P])
_factor_ws_bytes = _sig("kfac_factor_ws_bytes", [ctypes.POINTER(LayerDesc), _i32, _i32, _pi64])
_factor_all = _sig("kfac_factor_all", [_P, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.c_int, _pf32, _pf32, _P, _P, _P])
_reduce_scatter = _sig("kfac_reduce_scatter_factors", [_P, _P, _P, _P, _P])
_damped_inverse = _sig("kfac_damped_inverse", [_P, _i32, _P, _f32, _P, _P, _P, _P, _P])
_precondition = _sig("kfac_precondition", [_P, _i32, _P, _P, _P, _P, _P])
_allgather = _sig("kfac_allgather_precond", [_P, _P, _P, _P])
_plan_create_stale = _sig("kfac_plan_create_stale", [_P, ctypes.POINTER(_P)])
_plan_is_stale = _sig("kfac_plan_is_stale", [_P])
_plan_create_grefresh = _sig("kfac_plan_create_grefresh", [_P, ctypes.POINTER(_P)])
_plan_refresh_kind = _sig("kfac_plan_refresh_kind", [_P])
_refresh_interval = _sig("kfac_refresh_interval", [_i32, _i32])
_refresh = _sig("kfac_refresh", [_i64, _i32, _i32, _i64, _i32])
_factor_diff = _sig("kfac_factor_diff", [_P, _i32, _P, _P, _P, _P, _P])
RAMPUP, STEP13 = 0, 1
_bn_grads = _sig("kfac_bn_grads", [_i32, _pi32, _pi32, ctypes.POINTER(_P), ctypes.POINTER(_P), ctypes.c_int, _i32,
                                    ctypes.POINTER(_P)])
_bn_precondition = _sig("kfac_bn_precondition", [_i32, _pi32, _i32, ctypes.POINTER(_P), ctypes.POINTER(_P), _f32, _i32,
                                                  ctypes.POINTER(_P), _P, _i64, _P])
_bn_exchange = _sig("kfac_bn_exchange", [_P, _i32, _pi32, _i32, ctypes.POINTER(_P), ctypes.POINTER(_P),
                                          ctypes.POINTER(_P), _P])
_bn_ws_bytes = _sig("kfac_bn_ws_bytes", [_i32, _pi32, _i32, _pi64])
_set_inv_prec = _sig("kfac_plan_set_inverse_precision", [_P, _i32])
_inv_report = _sig("kfac_inverse_report", [_P, _i32, _P, ctypes.POINTER(ctypes.c_double), _pi32, _P])
INV_AUTO, INV_FP64, INV_INT8 = 0, 1, 2
_set_rs_mode = _sig("kfac_plan_set_rs_mode", [_P, _i32])
RS_PADDED, RS_PER_OWNER = 0, 1
_set_wire = _sig("kfac_plan_set_wire", [_P, _i32, _f32, _f32])
WIRE_FP32, WIRE_FP16 = 0, 1
_reduce_scatter_ws = _sig("kfac_reduce_scatter_factors_ws", [_P, _P, _P, _P, _P, _P])
_update = _sig("kfac_update", [_P, _P, ctypes.POINTER(_P), ctypes.POINTER(_P), _f32, _f32, _i32, _f32, _P, _P])

EXPORTS = ["kfac_last_error", "kfac_version", "kfac_launch_count", "kfac_plan_create", "kfac_plan_query", "kfac_plan_rank_layers",
           "kfac_plan_destroy", "kfac_comm_unique_id", "kfac_comm_create", "kfac_comm_destroy", "kfac_factor_A",
           "kfac_factor_G", "kfac_factor_ws_bytes", "kfac_factor_all", "kfac_reduce_scatter_factors",
           "kfac_damped_inverse", "kfac_precondition", "kfac_allgather_precond", "kfac_plan_create_stale",
           "kfac_plan_is_stale", "kfac_refresh_interval", "kfac_refresh", "kfac_factor_diff", "kfac_update", "kfac_bn_grads",
           "kfac_bn_precondition", "kfac_bn_ws_bytes", "kfac_bn_exchange",
           "kfac_plan_create_grefresh", "kfac_plan_refresh_kind", "kfac_plan_set_inverse_precision",
           "kfac_inverse_report", "kfac_plan_set_rs_mode", "kfac_plan_set_wire", "kfac_reduce_scatter_factors_ws"]


def _check(st, where):
    if st != 0:
        raise KfacError(st, where)


def version() -> str:
    return _lib.kfac_version().decode()


def launch_count() -> int:
    """Kernels launched by libkfac.so in this process (instrumentation)."""
    return int(_lib.kfac_launch_count())


def _ptr(t):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        return t
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


# ------------------------------------------------------------------ plan
class Plan:
    """kfac_plan_create / _query / _rank_layers / _destroy."""

    def __init__(self, layers, world, n_local, policy=RR, stale_of=None, grefresh_of=None):
        self.layers = list(layers)
        h = _P()
        if stale_of is not None:  # kfac_plan_create_stale: the dW-only layout of `stale_of`
            _check(_plan_create_stale(stale_of.h, ctypes.byref(h)), "kfac_plan_create_stale")
        elif grefresh_of is not None:  # kfac_plan_create_grefresh: the [dW, G] layout
            _check(_plan_create_grefresh(grefresh_of.h, ctypes.byref(h)), "kfac_plan_create_grefresh")
        else:
            arr = (LayerDesc * len(layers))(*[layer_desc(l) for l in layers])
            _check(_plan_create(arr, len(layers), int(world), int(n_local), int(policy), ctypes.byref(h)),
                   "kfac_plan_create")
        self.h = h
        self.stale = bool(_plan_is_stale(h))
        self.kind = int(_plan_refresh_kind(h))  # 0 full, 1 G refresh, 2 stale
        self.world, self.n_local, self.L = int(world), int(n_local), len(layers)
        self._q = None

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and _lib is not None:
            _lib.kfac_plan_destroy(h)
            self.h = None

    def query(self):
        if self._q is None:
            L = self.L
            owner = (ctypes.c_int32 * L)()
            seg = (ctypes.c_int64 * (3 * L))()
            ag = (ctypes.c_int64 * L)()
            rs_chunk, ag_chunk, ws = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
            _check(_plan_query(self.h, owner, seg, ctypes.byref(rs_chunk), ag, ctypes.byref(ag_chunk),
                               ctypes.byref(ws)), "kfac_plan_query")
            self._q = dict(owner=list(owner), seg_off=[list(seg[3 * l:3 * l + 3]) for l in range(L)],
                           rs_chunk=rs_chunk.value, ag_off=list(ag), ag_chunk=ag_chunk.value, ws_bytes=ws.value)
        return self._q

    def rank_layers(self, rank):
        L = self.L
        n = ctypes.c_int32()
        layers = (ctypes.c_int32 * L)()
        loc = (ctypes.c_int64 * (3 * L))()
        inv = (ctypes.c_int64 * (2 * L))()
        nf = ctypes.c_int64()
        _check(_plan_rank_layers(self.h, int(rank), ctypes.byref(n), layers, loc, inv, ctypes.byref(nf)),
               "kfac_plan_rank_layers")
        k = n.value
        return dict(layers=list(layers[:k]), local_off=[list(loc[3 * i:3 * i + 3]) for i in range(k)],
                    inv_off=[list(inv[2 * i:2 * i + 2]) for i in range(k)], inv_floats=nf.value)


    def set_inverse_precision(self, mode):
        """kfac_plan_set_inverse_precision: INV_AUTO (per-matrix bound), INV_FP64 or INV_INT8."""
        _check(_set_inv_prec(self.h, int(mode)), "kfac_plan_set_inverse_precision")

    def set_rs_mode(self, mode):
        """kfac_plan_set_rs_mode: RS_PADDED (one ReduceScatter) or RS_PER_OWNER (grouped per-owner Reduce)."""
        _check(_set_rs_mode(self.h, int(mode)), "kfac_plan_set_rs_mode")

    def set_wire(self, wire, scale_A=1.0, scale_G=1.0):
        """kfac_plan_set_wire: WIRE_FP32 or WIRE_FP16 (factor segments as fp16 x power-of-two scale).
        Changes ws_bytes: query the plan afterwards."""
        _check(_set_wire(self.h, int(wire), float(scale_A), float(scale_G)), "kfac_plan_set_wire")

    def stale_plan(self):
        """kfac_plan_create_stale: the plan of the steps that reuse stale factors."""
        return Plan(self.layers, self.world, self.n_local, stale_of=self)

    def grefresh_plan(self):
        """kfac_plan_create_grefresh: the plan of the steps that refresh G only."""
        return Plan(self.layers, self.world, self.n_local, grefresh_of=self)


def refresh_interval(schedule, epoch):
    return int(_refresh_interval(int(schedule), int(epoch)))


def refresh(t, epoch, schedule=RAMPUP, fresh_floor=500, interval=0):
    r = int(_refresh(int(t), int(epoch), int(schedule), int(fresh_floor), int(interval)))
    if r < 0:
        raise ValueError("kfac_refresh: bad argument (t < 0 or unknown schedule)")
    return bool(r)


# ------------------------------------------------------------------ comm
class Comm:
    def __init__(self, uid: bytes, rank: int, world: int, device: int):
        h = _P()
        _check(_comm_create(uid, int(rank), int(world), int(device), ctypes.byref(h)), "kfac_comm_create")
        self.h, self.rank, self.world = h, rank, world

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value and _lib is not None:
            _lib.kfac_comm_destroy(h)
            self.h = None


def comm_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(_comm_unique_id(buf), "kfac_comm_unique_id")
    return buf.raw


# ------------------------------------------------------------------ stages
def factor_ws_bytes(layer, n, which):
    b = ctypes.c_int64()
    _check(_factor_ws_bytes(ctypes.byref(layer_desc(layer)), int(n), int(which), ctypes.byref(b)),
           "kfac_factor_ws_bytes")
    return b.value


def factor_A(layer, x, n, alpha, out, ws=None, stream=None):
    _check(_factor_A(ctypes.byref(layer_desc(layer)), _ptr(x), _DT[x.dtype], int(n), float(alpha), _ptr(out),
                     _ptr(ws), ws.numel() * ws.element_size() if ws is not None else 0, _stream(stream)),
           "kfac_factor_A")


def factor_G(layer, gy, n, alpha, out, ws=None, stream=None):
    _check(_factor_G(ctypes.byref(layer_desc(layer)), _ptr(gy), _DT[gy.dtype], int(n), float(alpha), _ptr(out),
                     _ptr(ws), ws.numel() * ws.element_size() if ws is not None else 0, _stream(stream)),
           "kfac_factor_G")


def factor_all(plan, xs, gys, rs_send, ws, alphaA=None, alphaG=None, stream=None):
    L = plan.L
    if plan.stale:  # no factors on a stale step: only the redundant owners' dW copies
        _check(_factor_all(plan.h, None, None, 0, None, None, _ptr(rs_send), _ptr(ws), _stream(stream)),
               "kfac_factor_all")
        return
    xa = (_P * L)(*[x.data_ptr() for x in xs]) if xs is not None else None  # None: a G refresh
    ga = (_P * L)(*[g.data_ptr() for g in gys])
    aA = (ctypes.c_float * L)(*alphaA) if alphaA is not None else None
    aG = (ctypes.c_float * L)(*alphaG) if alphaG is not None else None
    _check(_factor_all(plan.h, xa, ga, _DT[gys[0].dtype], aA, aG, _ptr(rs_send), _ptr(ws), _stream(stream)),
           "kfac_factor_all")


def reduce_scatter_factors(comm, plan, rs_send, rs_recv, stream=None, ws=None):
    """kfac_reduce_scatter_factors, or kfac_reduce_scatter_factors_ws when `ws` is given (fp16 wire)."""
    c = comm.h if comm is not None else None
    if ws is None:
        _check(_reduce_scatter(c, plan.h, _ptr(rs_send), _ptr(rs_recv), _stream(stream)), "kfac_reduce_scatter_factors")
    else:
        _check(_reduce_scatter_ws(c, plan.h, _ptr(rs_send), _ptr(rs_recv), _ptr(ws), _stream(stream)),
               "kfac_reduce_scatter_factors_ws")


def damped_inverse(plan, rank, rs_recv, gamma, inv_ws, dev_status, pi_out, ws, stream=None):
    _check(_damped_inverse(plan.h, int(rank), _ptr(rs_recv), float(gamma), _ptr(inv_ws), _ptr(dev_status),
                           _ptr(pi_out), _ptr(ws), _stream(stream)), "kfac_damped_inverse")


def inverse_report(plan, rank, ws, n_owned, stream=None):
    """kfac_inverse_report (synchronises the stream): per owned matrix (A_d, G_d of each layer),
    the condition bound tr(M_d)/delta and the update precision (5 = int8 digits, 0 = fp64)."""
    bound = (ctypes.c_double * (2 * n_owned))()
    sl = (ctypes.c_int32 * (2 * n_owned))()
    _check(_inv_report(plan.h, int(rank), _ptr(ws), bound, sl, _stream(stream)), "kfac_inverse_report")
    return list(bound), list(sl)


def precondition(plan, rank, rs_recv, inv_ws, ag_buf, ws, stream=None):
    _check(_precondition(plan.h, int(rank), _ptr(rs_recv), _ptr(inv_ws), _ptr(ag_buf), _ptr(ws), _stream(stream)),
           "kfac_precondition")


def allgather_precond(comm, plan, ag_buf, stream=None):
    _check(_allgather(comm.h if comm is not None else None, plan.h, _ptr(ag_buf), _stream(stream)),
           "kfac_allgather_precond")


def factor_diff(plan, rank, recv_cur, recv_prev, diff, ws, stream=None):
    """kfac_factor_diff: Diff of every owned A, G between two refreshes, fp64 [2 * n_owned]."""
    _check(_factor_diff(plan.h, int(rank), _ptr(recv_cur), _ptr(recv_prev), _ptr(diff), _ptr(ws), _stream(stream)),
           "kfac_factor_diff")


def update(plan, ag_buf, ws_, w_prev, lr, momentum, ws, rescale=True, eps=1e-9, stream=None):
    """kfac_update: Eq. paramupdate + Normalizing Weights for every layer, in place."""
    L = plan.L
    wa = (_P * L)(*[_ptr(t).value for t in ws_])
    pa = (_P * L)(*[_ptr(t).value for t in w_prev])
    _check(_update(plan.h, _ptr(ag_buf), wa, pa, float(lr), float(momentum), 1 if rescale else 0, float(eps), _ptr(ws),
                   _stream(stream)), "kfac_update")


def _parr(ts):
    return (_P * len(ts))(*[_ptr(t).value for t in ts])


def bn_grads(c, hw, xhat, gy, n, S, stream=None):
    """kfac_bn_grads: per-sample BN scale / shift gradients S[l] [n, 2C] (NEXT-2, R-22)."""
    nl = len(c)
    _check(_bn_grads(nl, (ctypes.c_int32 * nl)(*c), (ctypes.c_int32 * nl)(*hw), _parr(xhat), _parr(gy),
                     _DT[xhat[0].dtype], int(n), _parr(S), _stream(stream)), "kfac_bn_grads")


def bn_ws_bytes(c, n):
    nl = len(c)
    b = ctypes.c_int64()
    _check(_bn_ws_bytes(nl, (ctypes.c_int32 * nl)(*c), int(n), ctypes.byref(b)), "kfac_bn_ws_bytes")
    return b.value


def bn_precondition(c, n, S, grad, gamma_bn, full, out, ws=None, stream=None):
    """kfac_bn_precondition: (F + gamma_bn I)^-1 grad (full, Woodbury; ws of bn_ws_bytes) or the diagonal."""
    nl = len(c)
    wsb = ws.numel() * ws.element_size() if ws is not None else 0
    _check(_bn_precondition(nl, (ctypes.c_int32 * nl)(*c), int(n), _parr(S), _parr(grad), float(gamma_bn),
                            1 if full else 0, _parr(out), _ptr(ws), wsb, _stream(stream)), "kfac_bn_precondition")


def bn_exchange(comm, c, n_local, S_local, S_all, grad, stream=None):
    """kfac_bn_exchange: AllGather of the per-sample BN gradients, mean AllReduce of the BN grads."""
    nl = len(c)
    _check(_bn_exchange(comm.h, nl, (ctypes.c_int32 * nl)(*c), int(n_local), _parr(S_local), _parr(S_all), _parr(grad),
                        _stream(stream)), "kfac_bn_exchange")
