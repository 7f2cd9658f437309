"""oracle — TEST INFRASTRUCTURE ONLY (see oracle/oracle.c for the C part).

Plain, slow, obviously correct CPU reference for everything the hot path
computes.  It is cold: it never implements a warm-start step.  After any graph
update the expected result is simply the APSP matrix of the mutated graph
(PAPER.md P:38-52), computed here from scratch by Floyd–Warshall or
Dijkstra.  The definitional predicates of the paper's intermediate
products (need_update_list, Cost, candidate_node_list) are written out in
numpy exactly as the paper states them, so tests can compare the GPU
detection / candidate kernels set-for-set.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline and
``--impl reference`` legs may import this package.  It shares no code with
``paper_2412_15122_b200`` and never imports it.

Numerics: integer weights in int64 (INF sentinel of the int32 API mapped to
2^62), floating weights in fp64 (Q1, Q16).

Pins (tests/test_oracle.py): brute-force simple-path enumeration (n <= 7),
FW == Dijkstra, closed forms (cycle, path, star, uniform complete graph, line
metric, grid), the SPEC/paper worked examples in tests/golden/.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

INF64 = np.int64(1) << 62          # oracle-side integer infinity
API_INF_I32 = 0x3FFFFFFF           # the int32 API's absent/unreachable value (apsp_warm.h)


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        i64, vp = ctypes.c_int64, ctypes.c_void_p
        L.oracle_fw_i64.argtypes = [i64, vp, i64]
        L.oracle_fw_f64.argtypes = [i64, vp]
        L.oracle_fw_i64_pivots.argtypes = [i64, vp, i64, i64, i64]
        L.oracle_dijkstra_i64.argtypes = [i64, vp, i64, i64, i64, vp, vp]
        L.oracle_dijkstra_f64.argtypes = [i64, vp, i64, i64, vp, vp]
        L.oracle_dijkstra_rows_i64.argtypes = [i64, vp, i64, vp, i64, vp]
        L.oracle_dijkstra_rows_f64.argtypes = [i64, vp, vp, i64, vp]
        L.oracle_brute_i64.restype = i64
        L.oracle_brute_i64.argtypes = [i64, vp, i64, i64, i64]
        L.oracle_brute_f64.restype = ctypes.c_double
        L.oracle_brute_f64.argtypes = [i64, vp, i64, i64]
        L.oracle_dijkstra_rows_i32w.argtypes = [i64, vp, i64, ctypes.c_int32, i64, vp, i64, vp, ctypes.c_int]
        L.oracle_fw_minimax_i64.argtypes = [i64, vp, i64]
        L.oracle_fw_minimax_f64.argtypes = [i64, vp]
        L.oracle_brute_minimax_i64.restype = i64
        L.oracle_brute_minimax_i64.argtypes = [i64, vp, i64, i64, i64]
        L.oracle_count_shortest_i64.restype = i64
        L.oracle_count_shortest_i64.argtypes = [i64, vp, i64, i64, i64, i64]
        _lib = L
    return _lib


# ----------------------------------------------------------------------------
# representation helpers
# ----------------------------------------------------------------------------
def is_int(W) -> bool:
    return np.issubdtype(np.asarray(W).dtype, np.integer)


def to_oracle(W):
    """int32 API matrix -> int64 with INF64; fp32 -> fp64 (exact)."""
    W = np.asarray(W)
    if is_int(W):
        A = W.astype(np.int64)
        A[W >= API_INF_I32] = INF64
        return np.ascontiguousarray(A)
    return np.ascontiguousarray(W.astype(np.float64))


def from_oracle_i32(D64):
    """int64 distances -> int32 API values (INF64 -> INF).  A finite distance
    >= the API INF violates the API precondition (Q1)."""
    D64 = np.asarray(D64)
    fin = D64 < INF64
    if np.any(D64[fin] >= API_INF_I32):
        raise ValueError("finite distance >= APSP_INF_I32: outside the int32 API's range")
    out = np.where(fin, D64, API_INF_I32).astype(np.int32)
    return out


# ----------------------------------------------------------------------------
# cold APSP: Floyd–Warshall and Dijkstra
# ----------------------------------------------------------------------------
def fw(W):
    """APSP of W by plain Floyd–Warshall.  int -> int32 API values; float -> fp64."""
    A = to_oracle(W)
    n = A.shape[0]
    if is_int(W):
        lib().oracle_fw_i64(n, A.ctypes.data, int(INF64))
        return from_oracle_i32(A)
    lib().oracle_fw_f64(n, A.ctypes.data)
    return A


def fw_minimax(W):
    """All-pairs minimax (bottleneck) distances by FW with (+) -> max."""
    A = to_oracle(W)
    n = A.shape[0]
    if is_int(W):
        lib().oracle_fw_minimax_i64(n, A.ctypes.data, int(INF64))
        return from_oracle_i32(A)
    lib().oracle_fw_minimax_f64(n, A.ctypes.data)
    return A


def brute_minimax_apsp(W):
    """Exhaustive simple-path enumeration of the minimax distance (n <= 12)."""
    A = to_oracle(W)
    n = A.shape[0]
    out = np.zeros((n, n), np.int64)
    for s_ in range(n):
        for t in range(n):
            r = lib().oracle_brute_minimax_i64(n, A.ctypes.data, int(INF64), s_, t)
            out[s_, t] = API_INF_I32 if r >= INF64 else r
    return out.astype(np.int32)


def need_update_removal_minimax(D, k):
    """Theorem 4 with (+) -> max: pair (i, j) listed iff max(D[i][k], D[k][j]) == D[i][j]."""
    A = to_oracle(D)
    lhs = np.maximum(A[:, k][:, None], A[k, :][None, :])
    m = (lhs == A) & _fin(A)
    m[k, :] = False
    m[:, k] = False
    np.fill_diagonal(m, False)
    return m


def fw_raw_i64(A64, k0, k1):
    """Run FW pivots [k0,k1) in place on an int64 oracle matrix (timing samples)."""
    lib().oracle_fw_i64_pivots(A64.shape[0], A64.ctypes.data, int(INF64), k0, k1)


def dijkstra_rows(W, srcs):
    """Rows srcs of the APSP matrix, by one Dijkstra per source."""
    A = to_oracle(W)
    n = A.shape[0]
    srcs = np.ascontiguousarray(np.asarray(srcs, np.int64))
    if is_int(W):
        out = np.empty((len(srcs), n), np.int64)
        lib().oracle_dijkstra_rows_i64(n, A.ctypes.data, int(INF64), srcs.ctypes.data, len(srcs), out.ctypes.data)
        return from_oracle_i32(out)
    out = np.empty((len(srcs), n), np.float64)
    lib().oracle_dijkstra_rows_f64(n, A.ctypes.data, srcs.ctypes.data, len(srcs), out.ctypes.data)
    return out


def dijkstra_cols(W, dsts):
    """Columns dsts of the APSP matrix (Dijkstra on the reversed graph W^T)."""
    return dijkstra_rows(np.ascontiguousarray(np.asarray(W).T), dsts).T


def dijkstra_rows_i32(W, srcs, reverse=False):
    """Rows (or, reverse=True, columns) srcs of the APSP matrix of an int32 W
    (API INF sentinel), by Dijkstra reading W in place: no int64 copy of W."""
    W = np.asarray(W)
    assert W.dtype == np.int32 and W.strides[1] == 4
    n = W.shape[0]
    srcs = np.ascontiguousarray(np.asarray(srcs, np.int64))
    out = np.empty((len(srcs), n), np.int64)
    lib().oracle_dijkstra_rows_i32w(n, W.ctypes.data, W.strides[0] // 4, API_INF_I32, int(INF64),
                                    srcs.ctypes.data, len(srcs), out.ctypes.data, int(reverse))
    return from_oracle_i32(out)


def dijkstra_pair(W, s, t):
    """(dist, path) for one pair by Dijkstra with early stop."""
    A = to_oracle(W)
    n = A.shape[0]
    pred = np.empty(n, np.int64)
    if is_int(W):
        dist = np.empty(n, np.int64)
        lib().oracle_dijkstra_i64(n, A.ctypes.data, int(INF64), s, t, dist.ctypes.data, pred.ctypes.data)
        d = dist[t]
        if d >= INF64:
            return API_INF_I32, []
    else:
        dist = np.empty(n, np.float64)
        lib().oracle_dijkstra_f64(n, A.ctypes.data, s, t, dist.ctypes.data, pred.ctypes.data)
        d = dist[t]
        if not np.isfinite(d):
            return np.inf, []
    path = [t]
    while path[-1] != s:
        path.append(int(pred[path[-1]]))
    return d, path[::-1]


def brute(W, s, t):
    """Minimum over all simple s->t paths by exhaustive enumeration (n <= 12)."""
    A = to_oracle(W)
    n = A.shape[0]
    assert n <= 12
    if is_int(W):
        r = lib().oracle_brute_i64(n, A.ctypes.data, int(INF64), s, t)
        return API_INF_I32 if r >= INF64 else int(r)
    return lib().oracle_brute_f64(n, A.ctypes.data, s, t)


def brute_apsp(W):
    n = np.asarray(W).shape[0]
    dt = np.int64 if is_int(W) else np.float64
    out = np.zeros((n, n), dt)
    for s in range(n):
        for t in range(n):
            out[s, t] = brute(W, s, t)
    return out.astype(np.int32) if is_int(W) else out


def count_shortest(W, s, t, dist):
    A = to_oracle(W)
    return int(lib().oracle_count_shortest_i64(A.shape[0], A.ctypes.data, int(INF64), s, t, int(dist)))


# ----------------------------------------------------------------------------
# definitional predicates of the paper's intermediate products
# ----------------------------------------------------------------------------
def _fin(D):
    return D < INF64 if is_int(D) else np.isfinite(D)


def _eq(lhs, D, tau):
    """The paper's '=' test.  Integers: exact.  Floats: lhs <=
    D*(1+tau) (Q4: conservative, ties go to 'needs update')."""
    if is_int(D):
        return lhs == D
    return lhs <= D * (1.0 + tau)


def need_update_removal(D, k, tau=1e-5):
    """need_update_list of removing node k (Theorem 4 P:381-407 /
    Corollary 3 P:409-433): pair (i, j), i, j != k, is listed iff
    SPD(i,j|G) = SPD(i,k|G) + SPD(k,j|G).  Unreachable pairs (D = INF) are
    never listed (Q5).  i == j is never listed (D[i][i] = 0 stays 0).
    Returns an n x n boolean mask in pre-removal indexing."""
    A = to_oracle(D)
    n = A.shape[0]
    lhs = A[:, k][:, None] + A[k, :][None, :]
    m = _eq(lhs, A, tau) & _fin(A)
    m[k, :] = False
    m[:, k] = False
    np.fill_diagonal(m, False)
    return m


def need_update_increase(D, u, v, w_old, directed=True, tau=1e-5):
    """Pairs whose shortest path may use edge (u, v) of weight w_old: the edge
    analogue of Theorem 4: listed iff D[i][u] + w_old + D[v][j] =
    D[i][j] (undirected: either orientation).  Never INF pairs, never i == j."""
    A = to_oracle(D)
    w = np.int64(w_old) if is_int(D) else np.float64(w_old)
    lhs = A[:, u][:, None] + w + A[v, :][None, :]
    m = _eq(lhs, A, tau)
    if not directed:
        lhs2 = A[:, v][:, None] + w + A[u, :][None, :]
        m |= _eq(lhs2, A, tau)
    m &= _fin(A)
    np.fill_diagonal(m, False)
    return m


def cost(mask, N):
    """Definition 1 (Eq. equ:cost_defi): C = Phi / (N - 1), Phi =
    number of sources with a non-empty need_update_list."""
    phi = int(np.count_nonzero(mask.any(axis=1)))
    return phi, phi / (N - 1)


def candidates(D, s, t, tau=1e-5):
    """candidate_node_list of alg:sp_apsp by Theorem 4: nodes k
    with SPD(s,k) + SPD(k,t) = SPD(s,t); empty if t is unreachable."""
    A = to_oracle(D)
    if not _fin(A[s, t]):
        return np.zeros(0, np.int64)
    lhs = A[s, :] + A[:, t]
    return np.nonzero(_eq(lhs, A[s, t], tau) & _fin(lhs))[0]


def path_weight(W, path):
    A = to_oracle(W)
    tot = A.dtype.type(0)
    for a, b in zip(path[:-1], path[1:]):
        tot = tot + A[a, b]
    return tot


def path_is_valid(W, path, s, t):
    """Starts at s, ends at t, no repeated node, every hop a present edge."""
    if not path or path[0] != s or path[-1] != t or len(set(path)) != len(path):
        return False
    A = to_oracle(W)
    return all(_fin(A[a, b]) for a, b in zip(path[:-1], path[1:]))


# ----------------------------------------------------------------------------
# APSP-matrix invariants: diag 0, triangle inequality, D <= W
# ----------------------------------------------------------------------------
def check_invariants(D, W, directed=True, rtol=0.0):
    A, Wo = to_oracle(D), to_oracle(W)
    n = A.shape[0]
    assert np.all(np.diag(A) == 0)
    if is_int(A):
        assert np.all(A <= Wo)
    else:
        assert np.all(A <= Wo * (1 + rtol))
    for k in range(n):
        tri = A[:, k][:, None] + A[k, :][None, :]
        if is_int(A):
            assert np.all(A <= tri)
        else:
            assert np.all(A <= tri * (1 + rtol) + 0.0)
    if not directed:
        assert np.array_equal(A, A.T)
