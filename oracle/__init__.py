"""fp64 CPU oracle for the distributed K-FAC hot path (arXiv 1811.12019).

TEST INFRASTRUCTURE ONLY -- only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this package.  It shares no
code with the CUDA path (paper_1811_12019_b200/) and neither imports the other;
the only common module is ``synth`` (shape tables + seeded inputs, no K-FAC
arithmetic).

Arithmetic lives in ``kfac_oracle.c`` (plain fp64 loops, built with gcc by
``build()``); this module marshals arguments and implements the host-side
parts of the method in plain Python:

* ``plan``             layer ownership + wire layout (
                       readings R-15, R-16) -- an implementation independent
                       of the library's plan.cpp, compared bit-exactly.
* ``reduce_scatter``   ReduceScatterV(mean) simulated in-process, summation in
                       ascending rank order then x 1/P (R-11);
                       optionally with the fp16 factor wire (``wire_fp16``,
                       NEXT-4(ii), reading R-23).
* ``all_gather``       AllGatherV of the primary owners' 𝒢.
* ``damping_schedule`` warmup damping recurrence (reading R-2).
* ``kfac_step``        Algorithm 1's body minus fwd/bwd/update.
* ``refresh_interval`` / ``refresh`` / ``refresh_kinds`` / ``fim_diff`` /
  ``diff_percentiles`` / ``stale_results`` / ``grefresh_results`` and
  ``plan(stale=True | g_only=True)``: stale Fisher information
  (NEXT-1; reading R-20).
* ``learning_rate`` / ``momentum`` / ``apply_update`` / ``rescale_weights`` /
  ``update_layer``: the update after the AllGather (NEXT-3; R-21).
* ``bn_sample_grads`` / ``bn_fisher`` / ``bn_precondition``: the Batch
  Normalization Fisher, full and diagonal (NEXT-2; P:493-494, P:665-668,
  P:740-763; R-22).

Parity status: every function here is pinned by tests/test_oracle_*.py (see
DESIGN.md §Oracle pins); none is "parity unpinned".
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "kfac_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

FMT = {"bf16": 0, "fp16": 1}


def build(force: bool = False) -> str:
    """Compile kfac_oracle.c -> liboracle.so with gcc (fp64, OpenMP, no FP contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", _LIB + ".tmp", _SRC, "-lm"]
        subprocess.check_call(cmd)
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB)
        i32, i64, f64 = ctypes.c_int, ctypes.c_int64, ctypes.c_double
        P = ctypes.c_void_p
        L.or_decode_half.argtypes = [ctypes.c_uint16, i32]
        L.or_decode_half.restype = f64
        L.or_factor_A.argtypes = [i32] * 11 + [P, i32, f64, P, i32]
        L.or_factor_A_entries.argtypes = [i32] * 11 + [P, i32, f64, P, i64, P, i32]
        L.or_factor_G.argtypes = [i64, i32, P, i32, f64, P, i32]
        L.or_factor_G_entries.argtypes = [i64, i32, P, i32, f64, P, i64, P, i32]
        L.or_pack_upper.argtypes = [P, i32, P]
        L.or_unpack_upper.argtypes = [P, i32, P]
        L.or_damp.argtypes = [P, i32, P, i32, f64, P]
        L.or_cholesky.argtypes = [P, i32, P, i32]
        L.or_tri_inv_lower.argtypes = [P, i32, P, i32]
        L.or_inverse_spd.argtypes = [P, i32, P, i32]
        L.or_precondition.argtypes = [P, i32, P, i32, P, P, i32]
        L.or_precondition_entries.argtypes = [P, i32, P, i32, P, P, i64, P, i32]
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().or_max_threads())


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


# --------------------------------------------------------------------------
# geometry (plain definitions, written here independently of the library)
# --------------------------------------------------------------------------
def out_hw(layer):
    if layer["kind"] == 1:
        return 1, 1
    ho = (layer["h_in"] + 2 * layer["pad_h"] - layer["kh"]) // layer["stride_h"] + 1
    wo = (layer["w_in"] + 2 * layer["pad_w"] - layer["kw"]) // layer["stride_w"] + 1
    return ho, wo


def dims(layer):
    return layer["c_in"] * layer["kh"] * layer["kw"] + (1 if layer["has_bias"] else 0), layer["c_out"]


def rows(layer, n):
    ho, wo = out_hw(layer)
    return n * ho * wo


def _geom(layer):
    if layer["kind"] == 1:
        return (1, 1, layer["c_in"], 1, 1, 1, 1, 0, 0)
    return (layer["h_in"], layer["w_in"], layer["c_in"], layer["kh"], layer["kw"],
            layer["stride_h"], layer["stride_w"], layer["pad_h"], layer["pad_w"])


# --------------------------------------------------------------------------
# stages 1-2: Kronecker factors
# --------------------------------------------------------------------------
def factor_A(layer, x_bits, n, alpha=None, fmt="bf16", threads=0):
    """A = alpha * Σ_rows ã ãᵀ (full, fp64). Default alpha = 1/rows (R-3)."""
    d_a, _ = dims(layer)
    if alpha is None:
        alpha = 1.0 / rows(layer, n)
    x = _c(x_bits, np.uint16)
    A = np.empty((d_a, d_a), dtype=np.float64)
    st = lib().or_factor_A(n, *_geom(layer), int(layer["has_bias"]), _p(x), FMT[fmt],
                           float(alpha), _p(A), threads)
    if st:
        raise ValueError("empty capture (S:201)")
    return A


def factor_A_entries(layer, x_bits, n, ij, alpha=None, fmt="bf16", threads=0):
    if alpha is None:
        alpha = 1.0 / rows(layer, n)
    x = _c(x_bits, np.uint16)
    ij = _c(ij, np.int64).reshape(-1, 2)
    out = np.empty(len(ij), dtype=np.float64)
    lib().or_factor_A_entries(n, *_geom(layer), int(layer["has_bias"]), _p(x), FMT[fmt],
                              float(alpha), _p(ij), len(ij), _p(out), threads)
    return out


def factor_G(gy_bits, n_rows, c, alpha=None, fmt="bf16", threads=0):
    """G = alpha * Σ_rows g gᵀ (full, fp64). Default alpha = 1/rows (R-3, R-4)."""
    if alpha is None:
        alpha = 1.0 / n_rows
    g = _c(gy_bits, np.uint16)
    G = np.empty((c, c), dtype=np.float64)
    if lib().or_factor_G(n_rows, c, _p(g), FMT[fmt], float(alpha), _p(G), threads):
        raise ValueError("empty capture (S:201)")
    return G


def factor_G_entries(gy_bits, n_rows, c, ij, alpha=None, fmt="bf16", threads=0):
    if alpha is None:
        alpha = 1.0 / n_rows
    g = _c(gy_bits, np.uint16)
    ij = _c(ij, np.int64).reshape(-1, 2)
    out = np.empty(len(ij), dtype=np.float64)
    lib().or_factor_G_entries(n_rows, c, _p(g), FMT[fmt], float(alpha), _p(ij), len(ij), _p(out), threads)
    return out


# --------------------------------------------------------------------------
# symmetric packing (R-10)
# --------------------------------------------------------------------------
def packed_len(d):
    return d * (d + 1) // 2


def pack(M):
    M = _c(M, np.float64)
    n = M.shape[0]
    if M.shape != (n, n):
        raise ValueError("pack: non-square input")
    if n and np.max(np.abs(M - M.T)) > 1e-12 * max(np.max(np.abs(M)), 1e-300):
        raise ValueError("pack: asymmetric input (S:36)")
    p = np.empty(packed_len(n), dtype=np.float64)
    lib().or_pack_upper(_p(M), n, _p(p))
    return p


def unpack(p):
    p = _c(p, np.float64)
    n = int((math.isqrt(8 * len(p) + 1) - 1) // 2)
    if packed_len(n) != len(p):
        raise ValueError("unpack: length is not d(d+1)/2")
    M = np.empty((n, n), dtype=np.float64)
    lib().or_unpack_upper(_p(p), n, _p(M))
    return M


# --------------------------------------------------------------------------
# stage 4: damping + inverse (P:466-473 R-1; P:247-260, P:328 R-12)
# --------------------------------------------------------------------------
def damp(A, G, gamma):
    A = _c(A, np.float64).copy()
    G = _c(G, np.float64).copy()
    pi = np.zeros(1)
    if lib().or_damp(_p(A), A.shape[0], _p(G), G.shape[0], float(gamma), _p(pi)):
        raise ValueError("damping requires gamma > 0 (S:217)")
    return A, G, float(pi[0])


def cholesky(M, threads=0):
    M = _c(M, np.float64)
    L = np.empty_like(M)
    st = lib().or_cholesky(_p(M), M.shape[0], _p(L), threads)
    return L, int(st)


def inverse(M, threads=0):
    """(X, status): X = M⁻¹ via Cholesky; status = 0 or failing pivot + 1."""
    M = _c(M, np.float64)
    X = np.zeros_like(M)
    st = lib().or_inverse_spd(_p(M), M.shape[0], _p(X), threads)
    return X, int(st)


# --------------------------------------------------------------------------
# stage 5: preconditioning (R-14)
# --------------------------------------------------------------------------
def precondition(Ginv, Ainv, dW, threads=0):
    Ginv, Ainv, dW = _c(Ginv, np.float64), _c(Ainv, np.float64), _c(dW, np.float64)
    dg, da = dW.shape
    if Ginv.shape != (dg, dg) or Ainv.shape != (da, da):
        raise ValueError("precondition: shape mismatch (S:72)")
    out = np.empty((dg, da), dtype=np.float64)
    lib().or_precondition(_p(Ginv), dg, _p(Ainv), da, _p(dW), _p(out), threads)
    return out


def precondition_entries(Ginv, Ainv, dW, ij, threads=0):
    Ginv, Ainv, dW = _c(Ginv, np.float64), _c(Ainv, np.float64), _c(dW, np.float64)
    dg, da = dW.shape
    ij = _c(ij, np.int64).reshape(-1, 2)
    out = np.empty(len(ij), dtype=np.float64)
    lib().or_precondition_entries(_p(Ginv), dg, _p(Ainv), da, _p(dW), _p(ij), len(ij), _p(out), threads)
    return out


# --------------------------------------------------------------------------
# schedules (Table 3; reading R-2)
# --------------------------------------------------------------------------
def damping_alpha(gamma0, gamma_target, t_warmup):
    """α = 2·log10(γ⁽⁰⁾/γ_target) / t_warmup."""
    if t_warmup <= 0:
        raise ValueError("t_warmup must be > 0")
    return 2.0 * math.log10(gamma0 / gamma_target) / t_warmup


def damping_schedule(gamma0, gamma_target, t_warmup, steps):
    """[γ⁽⁰⁾, γ⁽¹⁾, ...]: γ⁽ᵗ⁺¹⁾ = (1−α)γ⁽ᵗ⁾ + α·γ_target."""
    a = damping_alpha(gamma0, gamma_target, t_warmup)
    g = [float(gamma0)]
    for _ in range(steps):
        g.append((1.0 - a) * g[-1] + a * gamma_target)
    return g


# --------------------------------------------------------------------------
# a0: ownership + wire layout (R-15, R-16)
# --------------------------------------------------------------------------
POLICY_RR, POLICY_LPT = 0, 1
ALIGN = 16  # elements (64 B) per segment start


def _align(v):
    return (v + ALIGN - 1) // ALIGN * ALIGN


def layer_cost(layer):
    """Stage-4/5 cost model (R-15): dA³ + dG³ + 2dG²dA + 2dGdA²."""
    a, g = dims(layer)
    return a ** 3 + g ** 3 + 2 * g * g * a + 2 * g * a * a


def plan(layers, world, policy=POLICY_RR, stale=False, g_only=False):
    """Owner map and owner-major segment layout.

    owner[l]: primary owner.  RR: l mod P.  LPT: layers by (-cost, l), each to
    argmin (load, rank).  If P > L, rank r >= L also owns layer r mod L
    (redundant copy).  Rank r's chunk lists its owned layers ascending,
    each with segments [∇W (dG·dA), A packed, G packed], every segment start
    aligned to 16 elements; rs_chunk = max chunk.  AG: each rank's chunk holds
    its primary layers' 𝒢 (dG·dA) ascending, aligned; ag_chunk = max.

    stale=True: the wire layout of a step that reuses stale factors (P:701-704,
    "reduce the frequency of updating (A, G, F)"; reading R-20): the same
    owners, but each owned layer carries only its ∇W segment; the A and G
    offsets are None (seg_off -1).  The AG layout is unchanged.

    g_only=True: the layout of a step that refreshes G but keeps A stale
    (S:549): each owned layer carries [∇W, G packed]; A's offset is
    None (seg_off -1).
    """
    L, P = len(layers), int(world)
    if L < 1 or P < 1:
        raise ValueError("plan: L, P >= 1")
    if policy == POLICY_RR:
        owner = [l % P for l in range(L)]
    elif policy == POLICY_LPT:
        owner = [0] * L
        load = [0] * P
        for l in sorted(range(L), key=lambda l: (-layer_cost(layers[l]), l)):
            r = min(range(P), key=lambda r: (load[r], r))
            owner[l] = r
            load[r] += layer_cost(layers[l])
    else:
        raise ValueError("unknown policy")
    owned = [sorted([l for l in range(L) if owner[l] == r] + ([r % L] if r >= L else []))
             for r in range(P)]
    local = []  # per rank: {layer: (off_dw, off_a, off_g)} relative to the chunk
    chunk = []
    for r in range(P):
        off, m = 0, {}
        for l in owned[r]:
            a, g = dims(layers[l])
            o_w = off
            off = _align(off + g * a)
            if stale:
                m[l] = (o_w, None, None)
                continue
            if g_only:
                o_g = off
                off = _align(off + packed_len(g))
                m[l] = (o_w, None, o_g)
                continue
            o_a = off
            off = _align(off + packed_len(a))
            o_g = off
            off = _align(off + packed_len(g))
            m[l] = (o_w, o_a, o_g)
        local.append(m)
        chunk.append(off)
    rs_chunk = max(chunk)
    seg_off = np.zeros((L, 3), dtype=np.int64)
    for l in range(L):
        r = owner[l]
        seg_off[l] = [-1 if v is None else r * rs_chunk + v for v in local[r][l]]
    ag_local, ag_chunks = [], []
    for r in range(P):
        off, m = 0, {}
        for l in range(L):
            if owner[l] == r:
                a, g = dims(layers[l])
                m[l] = off
                off = _align(off + g * a)
        ag_local.append(m)
        ag_chunks.append(off)
    ag_chunk = max(ag_chunks)
    ag_off = np.array([owner[l] * ag_chunk + ag_local[owner[l]][l] for l in range(L)], dtype=np.int64)
    return dict(owner=np.array(owner, dtype=np.int32), owned=owned, local=local,
                seg_off=seg_off, rs_chunk=int(rs_chunk), ag_off=ag_off, ag_chunk=int(ag_chunk),
                world=P, L=L, stale=bool(stale), g_only=bool(g_only))


# --------------------------------------------------------------------------
# a4 / a8: simulated collectives (R-11, R-16)
# --------------------------------------------------------------------------
def wire_fp16(x, scale=1.0):
    """The fp16 wire value of x (NEXT-4(ii); reading R-9 of P:92-93, "half precision floating point
    numbers for both computation [and communication]"; R-23): x·scale rounded to the
    nearest IEEE binary16 value, ties to even (overflow to ±inf, gradual underflow), then ÷ scale.
    `scale` is a power of two, so both scalings are exact and only the rounding changes x."""
    s = float(scale)
    m, _ = math.frexp(s)
    if s <= 0 or m != 0.5:
        raise ValueError("wire scale must be a positive power of two")
    with np.errstate(over="ignore"):  # overflow to ±inf is the format's answer
        return np.asarray(np.asarray(x, dtype=np.float64) * s).astype(np.float16).astype(np.float64) / s


def _wire_mask(pl, n_elems):
    """Per element of one rank's send buffer: 0 = ∇W (fp32 on the wire), 1 = A, 2 = G."""
    P, c = pl["world"], pl["rs_chunk"]
    kind = np.zeros(P * c, dtype=np.int8)
    for r in range(P):
        for l, (o_w, o_a, o_g) in pl["local"][r].items():
            for k, o in ((1, o_a), (2, o_g)):
                if o is not None:
                    kind[r * c + o: r * c + o + packed_len(n_elems[l][k - 1])] = k
    return kind


def reduce_scatter(sends, pl, wire=None, layers=None):
    """ReduceScatterV(mean): rank r receives chunk r of Σ_{q=0..P-1} send_q (ascending), × 1/P.

    wire=(scale_A, scale_G) (NEXT-4(ii), R-23; needs `layers`): the factor segments travel as fp16 —
    every rank's A / G elements are replaced by wire_fp16(·, scale) and the owner takes the mean of
    the P wire values it receives (in fp64 here); ∇W travels in fp32 (exact mean)."""
    P, c = pl["world"], pl["rs_chunk"]
    if wire is not None:
        kind = _wire_mask(pl, [dims(L) for L in layers])
        sc = [None, float(wire[0]), float(wire[1])]
        sends = [np.asarray(s, dtype=np.float64).copy() for s in sends]
        for s in sends:
            for k in (1, 2):
                s[kind == k] = wire_fp16(s[kind == k], sc[k])
    acc = np.zeros(P * c, dtype=np.float64)
    for q in range(P):
        acc += np.asarray(sends[q], dtype=np.float64)
    acc *= 1.0 / P
    return [acc[r * c:(r + 1) * c].copy() for r in range(P)]


def all_gather(slots, pl):
    """AllGatherV: every rank receives the concatenation of every rank's AG chunk."""
    full = np.concatenate([np.asarray(s) for s in slots])
    return [full.copy() for _ in range(pl["world"])]


# --------------------------------------------------------------------------
# Algorithm 1 body: factors -> RS -> damp+invert -> precondition -> AG
# --------------------------------------------------------------------------
def build_send(layers, pl, rank, factors, dws):
    """Rank `rank`'s RS send buffer: (∇W, A packed, G packed) of every layer at every owner copy
    (∇W only for a stale plan; `factors` may then be None)."""
    P, c = pl["world"], pl["rs_chunk"]
    send = np.zeros(P * c, dtype=np.float64)
    for r in range(P):
        for l, (o_w, o_a, o_g) in pl["local"][r].items():
            a, g = dims(layers[l])
            base = r * c
            send[base + o_w: base + o_w + g * a] = np.asarray(dws[l], dtype=np.float64).reshape(-1)
            if o_g is None:  # stale layout: ∇W only
                continue
            A, G = factors[l]
            if o_a is not None:  # (a G-refresh layout carries no A)
                send[base + o_a: base + o_a + packed_len(a)] = pack(A)
            send[base + o_g: base + o_g + packed_len(g)] = pack(G)
    return send


def owned_results(layers, pl, rank, recv, gamma, threads=0):
    """Stages 4-5 on one rank: {layer: dict(A_d, G_d, pi, Ainv, Ginv, precond, status)}."""
    out = {}
    for l, (o_w, o_a, o_g) in pl["local"][rank].items():
        a, g = dims(layers[l])
        dW = recv[o_w:o_w + g * a].reshape(g, a)
        A = unpack(recv[o_a:o_a + packed_len(a)])
        G = unpack(recv[o_g:o_g + packed_len(g)])
        A_d, G_d, pi = damp(A, G, gamma)
        Ainv, sa = inverse(A_d, threads)
        Ginv, sg = inverse(G_d, threads)
        pre = precondition(Ginv, Ainv, dW, threads) if (sa == 0 and sg == 0) else None
        out[l] = dict(A=A, G=G, dW=dW, A_d=A_d, G_d=G_d, pi=pi, Ainv=Ainv, Ginv=Ginv,
                      precond=pre, status=(sa, sg))
    return out


def kfac_step(layers, rank_inputs, world, gamma, policy=POLICY_RR, fmt="bf16", threads=0, wire=None):
    """Simulate all P ranks.  rank_inputs[r] = (x_bits list, gy_bits list, dW list, n_local).
    wire: None (fp32 wire) or (scale_A, scale_G) of the fp16 factor wire (reduce_scatter).

    Returns dict(plan, sends, recvs, results (per rank), gathered (per rank AG buffer)).
    """
    pl = plan(layers, world, policy)
    sends = []
    for r in range(world):
        xs, gys, dws, n = rank_inputs[r]
        factors = []
        for l, layer in enumerate(layers):
            A = factor_A(layer, xs[l], n, fmt=fmt, threads=threads)
            rws = rows(layer, n)
            G = factor_G(gys[l], rws, layer["c_out"], fmt=fmt, threads=threads)
            factors.append((A, G))
        sends.append(build_send(layers, pl, r, factors, dws))
    recvs = reduce_scatter(sends, pl, wire=wire, layers=layers)
    results = [owned_results(layers, pl, r, recvs[r], gamma, threads) for r in range(world)]
    slots = []
    for r in range(world):
        slot = np.zeros(pl["ag_chunk"], dtype=np.float64)
        for l in range(len(layers)):
            if pl["owner"][l] == r:
                a, g = dims(layers[l])
                o = pl["ag_off"][l] - r * pl["ag_chunk"]
                slot[o:o + g * a] = results[r][l]["precond"].reshape(-1)
        slots.append(slot)
    gathered = all_gather(slots, pl)
    return dict(plan=pl, sends=sends, recvs=recvs, results=results, gathered=gathered)


# --------------------------------------------------------------------------
# NEXT-1: stale Fisher information
# --------------------------------------------------------------------------
def refresh_interval(epoch, schedule="rampup"):
    """interval⁽ᵉ⁾ of the epoch-e refresh schedule.

    "rampup": min(20, 5·⌊e/5⌋ + 1)            (the 10-minute run)
    "step13": 1 if e < 13 else 20             (the BN-diagonal study)
    """
    e = int(epoch)
    if e < 0:
        raise ValueError("epoch >= 0")
    if schedule == "rampup":
        return min(20, 5 * (e // 5) + 1)
    if schedule == "step13":
        return 1 if e < 13 else 20
    raise ValueError("unknown schedule")


def refresh(t, epoch, schedule="rampup", fresh_floor=500, interval=None):
    """Refresh decision of iteration t in epoch e: every iteration
    before `fresh_floor` ("after 500 iterations"), then when
    t mod interval⁽ᵉ⁾ = 0.  `interval` overrides the schedule (must be >= 1)."""
    iv = refresh_interval(epoch, schedule) if interval is None else int(interval)
    if iv < 1:
        raise ValueError("interval >= 1")
    return int(t) < int(fresh_floor) or int(t) % iv == 0


def fim_diff(X_cur, X_prev):
    """Diff⁽ᵗ⁾ = ‖X⁽ᵗ⁾ − X⁽ᵗ⁻¹⁾‖_F / ‖X⁽ᵗ⁻¹⁾‖_F of two full
    matrices, in fp64; None when ‖X⁽ᵗ⁻¹⁾‖_F = 0 ("recorded as missing")."""
    X_cur = np.asarray(X_cur, dtype=np.float64)
    X_prev = np.asarray(X_prev, dtype=np.float64)
    if X_cur.shape != X_prev.shape:
        raise ValueError("fim_diff: shapes differ")
    den = math.sqrt(float(np.sum(X_prev * X_prev)))
    if den == 0.0:
        return None
    D = X_cur - X_prev
    return math.sqrt(float(np.sum(D * D))) / den


def diff_percentiles(diffs, qs=(5, 25, 50, 75, 95)):
    """{5,25,50,75,95}th percentiles of the per-layer Diff values (Fig. 5
    caption), linear interpolation between order statistics; missing
    (None) values are dropped."""
    v = sorted(float(d) for d in diffs if d is not None)
    if not v:
        return {q: None for q in qs}
    out = {}
    for q in qs:
        pos = (len(v) - 1) * q / 100.0
        lo = int(math.floor(pos))
        hi = min(lo + 1, len(v) - 1)
        out[q] = v[lo] + (v[hi] - v[lo]) * (pos - lo)
    return out


def stale_results(layers, pl_stale, rank, recv, cached):
    """Stage 5 of a stale step on one rank: 𝒢 = G_d⁻¹ ∇W A_d⁻¹ with the cached
    inverses of the last refresh (`cached[l] = (Ainv, Ginv)`), ∇W from the
    stale-layout recv chunk (R-20)."""
    out = {}
    for l, (o_w, _, _) in pl_stale["local"][rank].items():
        a, g = dims(layers[l])
        dW = recv[o_w:o_w + g * a].reshape(g, a)
        Ainv, Ginv = cached[l]
        out[l] = dict(dW=dW, precond=precondition(Ginv, Ainv, dW))
    return out


# --------------------------------------------------------------------------
# NEXT-3: the update after the AllGather
# --------------------------------------------------------------------------
def learning_rate(eta0, e_start, e_end, p_decay, epoch):
    """η⁽ᵉ⁾ = η⁽⁰⁾·(1 − (e − e_start)/(e_end − e_start))^p_decay, clamped to η⁽⁰⁾
    before e_start and to 0 after e_end."""
    e = float(epoch)
    if e <= e_start:
        return float(eta0)
    if e >= e_end:
        return 0.0
    return float(eta0) * (1.0 - (e - e_start) / (e_end - e_start)) ** p_decay


def momentum(m0, eta0, eta_e):
    """m⁽ᵉ⁾ = (m⁽⁰⁾/η⁽⁰⁾)·η⁽ᵉ⁾."""
    return float(m0) / float(eta0) * float(eta_e)


def apply_update(w, w_prev, precond, eta, m):
    """Eq. paramupdate: w⁽ᵗ⁺¹⁾ = w⁽ᵗ⁾ − η·𝒢⁽ᵗ⁾ + m·(w⁽ᵗ⁾ − w⁽ᵗ⁻¹⁾), fp64.
    Returns (w⁽ᵗ⁺¹⁾, w⁽ᵗ⁾) -- the new weights and the new 'previous' weights."""
    w = np.asarray(w, dtype=np.float64)
    w_prev = np.asarray(w_prev, dtype=np.float64)
    precond = np.asarray(precond, dtype=np.float64)
    if w.shape != w_prev.shape or w.shape != precond.shape:
        raise ValueError("apply_update: shapes differ")
    return w - eta * precond + m * (w - w_prev), w.copy()


def rescale_weights(w, d_out, eps=1e-9):
    """Normalizing Weights: w ← √(2·d_out)·w/(‖w‖ + ε), ‖·‖ the Frobenius norm of the
    layer's weight tensor."""
    if int(d_out) < 1:
        raise ValueError("d_out >= 1")
    w = np.asarray(w, dtype=np.float64)
    return math.sqrt(2.0 * int(d_out)) * w / (math.sqrt(float(np.sum(w * w))) + eps)


def update_layer(w, w_prev, precond, eta, m, has_bias, rescale=True, eps=1e-9):
    """The whole post-AllGather update of one layer (reading R-21): Eq. paramupdate on the
    [d_out, dA] matrix [W | b] (𝒢 carries the bias column last, R-5), then Normalizing Weights on
    W only (the bias column is not rescaled), d_out = the layer's output channels."""
    w_new, w_keep = apply_update(w, w_prev, precond, eta, m)
    if rescale:
        nb = w_new.shape[1] - (1 if has_bias else 0)
        w_new = w_new.copy()
        w_new[:, :nb] = rescale_weights(w_new[:, :nb], w_new.shape[0], eps)
    return w_new, w_keep


# --------------------------------------------------------------------------
# NEXT-2: Fisher of the Batch Normalization layers (
# S:231-246; reading R-22).  Not factored into A and G: F is the empirical
# Fisher of the 2C parameters [scale γ_1..γ_C, shift β_1..β_C] of one BN layer.
# --------------------------------------------------------------------------
def _decode(bits, fmt):
    """Exact fp64 values of 16-bit bf16 / fp16 patterns."""
    b = np.ascontiguousarray(np.asarray(bits).reshape(-1)).view(np.uint16)
    if fmt == "bf16":
        return (b.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    if fmt == "fp16":
        return b.view(np.float16).astype(np.float64)
    raise ValueError("fmt: bf16 | fp16")


def bn_sample_grads(xhat_bits, gy_bits, n, hw, c, fmt="bf16"):
    """Per-sample BN parameter gradients S[s] = [Σ_p gy[s,p,:]·x̂[s,p,:], Σ_p gy[s,p,:]] (2C values,
    scale first then shift; y = γ·x̂ + β so ∂y/∂γ_c = x̂_c, ∂y/∂β_c = 1), p over the hw pixels of
    sample s, from the NHWC half-precision bit patterns the GPU consumes, in fp64."""
    x = _decode(xhat_bits, fmt).reshape(n, hw, c)
    g = _decode(gy_bits, fmt).reshape(n, hw, c)
    S = np.zeros((n, 2 * c), dtype=np.float64)
    for s in range(n):
        S[s, :c] = np.sum(g[s] * x[s], axis=0)
        S[s, c:] = np.sum(g[s], axis=0)
    return S


def bn_fisher(S, mode="full"):
    """F = (1/N) Σ_s S[s] S[s]ᵀ ("full", 2C x 2C) or its diagonal (1/N) Σ_s S[s]² ("diag",
    P:740-747 'approximate it with a diagonal matrix')."""
    S = np.asarray(S, dtype=np.float64)
    if mode == "full":
        F = np.zeros((S.shape[1], S.shape[1]), dtype=np.float64)
        for s in range(S.shape[0]):
            F += np.outer(S[s], S[s])
        return F / S.shape[0]
    if mode == "diag":
        return np.sum(S * S, axis=0) / S.shape[0]
    raise ValueError("mode: full | diag")


def bn_precondition(F, grad, gamma_bn):
    """(F + γ_BN·I)⁻¹·grad for a full F (via the oracle's Cholesky inverse), grad_i/(F_i + γ_BN) for a
    diagonal F; γ_BN = ρ_BN·γ."""
    if not gamma_bn > 0:
        raise ValueError("gamma_bn > 0")
    F = np.asarray(F, dtype=np.float64)
    grad = np.asarray(grad, dtype=np.float64)
    if F.ndim == 1:
        if F.shape != grad.shape:
            raise ValueError("bn_precondition: dimension mismatch")
        return grad / (F + gamma_bn)
    if F.shape != (grad.shape[0], grad.shape[0]):
        raise ValueError("bn_precondition: dimension mismatch")
    X, st = inverse(F + gamma_bn * np.eye(F.shape[0]))
    if st:
        raise ValueError("bn_precondition: F + gamma_bn I not positive definite")
    return X @ grad


def refresh_kinds(t, epoch, schedule="rampup", fresh_floor=500, a_multiple=1):
    """Per-kind refresh decision: G refreshes as ``refresh``; A with its interval
    multiplied by ``a_multiple`` ("refreshing A_{l-1} less frequently than G_l").
    Returns (refresh_A, refresh_G); A refreshing implies G refreshing."""
    if int(a_multiple) < 1:
        raise ValueError("a_multiple >= 1")
    iv = refresh_interval(epoch, schedule)
    rg = refresh(t, epoch, fresh_floor=fresh_floor, interval=iv)
    ra = refresh(t, epoch, fresh_floor=fresh_floor, interval=iv * int(a_multiple))
    return ra, rg


def grefresh_results(layers, pl_g, rank, recv, gamma, cached):
    """Stages 4-5 of a G-refresh step on one rank (R-20): G from the [∇W, G] recv chunk, damped with
    the cached π of the last full refresh, G_d = G + (√γ/π) I; A_d⁻¹ cached.  `cached[l] = (Ainv, pi)`."""
    out = {}
    for l, (o_w, _, o_g) in pl_g["local"][rank].items():
        a, g = dims(layers[l])
        dW = recv[o_w:o_w + g * a].reshape(g, a)
        G = unpack(recv[o_g:o_g + packed_len(g)])
        Ainv, pi = cached[l]
        G_d = G + (math.sqrt(gamma) / pi) * np.eye(g)
        Ginv, sg = inverse(G_d)
        pre = precondition(Ginv, Ainv, dW) if sg == 0 else None
        out[l] = dict(G=G, G_d=G_d, Ginv=Ginv, dW=dW, precond=pre, status=sg)
    return out
