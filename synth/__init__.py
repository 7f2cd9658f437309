"""synth — seeded synthetic inputs shared by the oracle side and the product side.

Holds NONE of the method's arithmetic (no relaxation, no min, no path sums):
only the counter-based weight generators of ``gen.c``,
the BASELINE.json workload recipes, and host-side index bookkeeping for
update sequences (add at index n, remove = swap-with-last; Q7/Q8).

Both ``oracle/`` and ``paper_2412_15122_b200/`` users (tests, bench.py) may
import this module; it imports neither of them.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gen.c")
_LIB = os.path.join(_HERE, "libsynth.so")

# The API's absent-edge sentinel for int32 (apsp_warm.h APSP_INF_I32). Kept as a
# plain constant here: the generator only writes it, it never computes with it.
INF_I32 = 0x3FFFFFFF


def build(force: bool = False) -> str:
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        u64, i64, i32, f64 = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int32, ctypes.c_double
        vp = ctypes.c_void_p
        L.synth_hash.restype = u64
        L.synth_hash.argtypes = [u64, u64, u64, u64]
        L.synth_uniform_int.restype = i64
        L.synth_uniform_int.argtypes = [u64, u64, u64, u64, i64, i64]
        L.synth_uniform01.restype = f64
        L.synth_uniform01.argtypes = [u64, u64, u64, u64]
        L.synth_graph_i32.argtypes = [u64, i64, ctypes.c_int, f64, ctypes.c_int, i64, i64, vp, i64, i32]
        L.synth_graph_f32.argtypes = [u64, i64, ctypes.c_int, f64, vp, i64, ctypes.c_float]
        L.synth_node_edges_i32.argtypes = [u64, u64, i64, ctypes.c_int, ctypes.c_int, i64, i64, vp, vp]
        L.synth_node_edges_f32.argtypes = [u64, u64, i64, ctypes.c_int, vp, vp]
        _lib = L
    return _lib


# ----------------------------------------------------------------------------
# Graph recipes
# ----------------------------------------------------------------------------
@dataclass(frozen=True)
class GraphSpec:
    """A synthetic dense graph recipe (one BASELINE.json config's graph)."""

    n: int
    directed: bool = True
    dtype: str = "i32"          # "i32" or "f32"
    density: float = 1.0
    kind: int = 0               # 0: U[lo,hi]; 1: log-uniform [lo,hi]; 2: fp32 grid (0,1]
    lo: int = 1
    hi: int = 100
    seed: int = 1


def graph(spec: GraphSpec, ld: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
    """Dense W (row-major, rows x ld) with W[i][j] = w(i->j), diag 0, absent = INF."""
    ld = spec.n if ld is None else ld
    L = lib()
    if spec.dtype == "i32":
        W = np.empty((spec.n, ld), np.int32) if out is None else out
        L.synth_graph_i32(spec.seed, spec.n, int(spec.directed), spec.density, spec.kind,
                          spec.lo, spec.hi, W.ctypes.data, W.strides[0] // 4, INF_I32)
    else:
        W = np.empty((spec.n, ld), np.float32) if out is None else out
        L.synth_graph_f32(spec.seed, spec.n, int(spec.directed), spec.density,
                          W.ctypes.data, W.strides[0] // 4, np.float32(np.inf))
    return W


def node_edges(spec: GraphSpec, t: int, n: int):
    """(out_w, in_w) of a node added at update index t to an n-node graph."""
    L = lib()
    if spec.dtype == "i32":
        o = np.empty(n, np.int32); i = np.empty(n, np.int32)
        L.synth_node_edges_i32(spec.seed, t, n, int(spec.directed), spec.kind, spec.lo, spec.hi,
                               o.ctypes.data, i.ctypes.data)
    else:
        o = np.empty(n, np.float32); i = np.empty(n, np.float32)
        L.synth_node_edges_f32(spec.seed, t, n, int(spec.directed), o.ctypes.data, i.ctypes.data)
    return o, i


def uniform_int(seed, stream, a, b, lo, hi) -> int:
    return int(lib().synth_uniform_int(seed, stream, a, b, lo, hi))


def uniform01(seed, stream, a, b) -> float:
    return float(lib().synth_uniform01(seed, stream, a, b))


# BASELINE.json configs (BJ.c1..c5) as graph recipes.  Full-size recipes; tests
# scale n down with dataclasses.replace(spec, n=...).
C1 = GraphSpec(n=256, directed=True, dtype="i32", kind=0, lo=1, hi=100)
C2 = GraphSpec(n=4096, directed=False, dtype="f32", kind=2)
C3 = GraphSpec(n=16384, directed=True, dtype="i32", density=0.9, kind=0, lo=1, hi=1000)
C4 = GraphSpec(n=32768, directed=True, dtype="i32", kind=0, lo=1, hi=1000)
C5 = GraphSpec(n=65536, directed=True, dtype="i32", kind=1, lo=1, hi=1_000_000)
CONFIGS = {"c1": C1, "c2": C2, "c3": C3, "c4": C4, "c5": C5}


# ----------------------------------------------------------------------------
# Host-side bookkeeping of W under the library's index convention
# ----------------------------------------------------------------------------
class HostGraph:
    """Host copy of W (cap x cap) mutated with the library's index convention:
    add -> new node at index n (Q8); remove k -> node n-1 moves into slot k
    (swap-with-last, Q7); undirected edits touch both directions (Q10).
    Pure bookkeeping: no distance arithmetic."""

    def __init__(self, W: np.ndarray, directed: bool, cap: int | None = None):
        n = W.shape[0]
        cap = n if cap is None else cap
        self.directed = directed
        self.dtype = W.dtype
        self.inf = INF_I32 if W.dtype == np.int32 else np.float32(np.inf)
        self.buf = np.full((cap, cap), self.inf, dtype=W.dtype)
        self.buf[:n, :n] = W[:n, :n]
        self.n = n

    @property
    def W(self) -> np.ndarray:
        return self.buf[: self.n, : self.n]

    def weight(self, u, v):
        return self.buf[u, v]

    def add_node(self, out_w, in_w) -> int:
        x = self.n
        assert x < self.buf.shape[0], "capacity"
        self.buf[x, :x] = out_w[:x]
        self.buf[:x, x] = in_w[:x]
        self.buf[x, x] = 0
        self.n += 1
        return x

    def remove_node(self, k) -> int:
        last = self.n - 1
        if k != last:
            self.buf[k, :] = self.buf[last, :]
            self.buf[:, k] = self.buf[:, last]
            self.buf[k, k] = 0
        self.buf[last, :] = self.inf
        self.buf[:, last] = self.inf
        self.n -= 1
        return last if k != last else -1

    def set_edge(self, u, v, w):
        self.buf[u, v] = w
        if not self.directed:
            self.buf[v, u] = w


def random_edge(seed: int, t: int, hg: HostGraph, stream: int = 5):
    """A uniformly random ordered pair u != v with a present edge (Q22)."""
    n = hg.n
    for r in range(1 << 20):
        u = uniform_int(seed, stream, t, 2 * r + 1, 0, n - 1)
        v = uniform_int(seed, stream, t, 2 * r + 2, 0, n - 2)
        v += v >= u
        if hg.weight(u, v) != hg.inf:
            return u, v
    raise RuntimeError("no present edge found")


def reweight_factor(seed: int, t: int) -> float:
    """f = 10^(2u-1), log-uniform in [0.1, 10] (Q18)."""
    return 10.0 ** (2.0 * uniform01(seed, 6, t, 0) - 1.0)


def new_weight(w_old, f, dtype):
    """Q18/Q20: int32 -> max(1, round-half-even(w*f)); fp32 -> fp32 product."""
    if dtype == np.int32:
        return int(max(1, np.rint(float(w_old) * f)))
    return np.float32(np.float32(w_old) * np.float32(f))


@dataclass
class Update:
    kind: str                 # "add" | "remove" | "reweight"
    t: int                    # update index (counter)
    k: int = -1               # remove
    u: int = -1               # reweight
    v: int = -1
    w_old: float = 0.0
    w_new: float = 0.0
    out_w: np.ndarray | None = None   # add
    in_w: np.ndarray | None = None
    n_before: int = 0


def update_sequence(spec: GraphSpec, hg: HostGraph, t0: int, count: int, with_vectors=True):
    """BJ.c4's sequence (Q18): update t has type t mod 3 in (add, remove, reweight).
    Mutates hg (bookkeeping) and returns the list of Update records."""
    seq = []
    for t in range(t0, t0 + count):
        n = hg.n
        typ = t % 3
        if typ == 0:
            o, i = node_edges(spec, t, n)
            up = Update("add", t, n_before=n, out_w=o if with_vectors else None,
                        in_w=i if with_vectors else None)
            hg.add_node(o, i)
        elif typ == 1:
            k = uniform_int(spec.seed, 5, t, 0, 0, n - 1)
            up = Update("remove", t, k=k, n_before=n)
            hg.remove_node(k)
        else:
            u, v = random_edge(spec.seed, t, hg)
            w_old = hg.weight(u, v)
            w_new = new_weight(w_old, reweight_factor(spec.seed, t), hg.dtype)
            up = Update("reweight", t, u=u, v=v, w_old=w_old, w_new=w_new, n_before=n)
            hg.set_edge(u, v, w_new)
        seq.append(up)
    return seq


def query_pairs(seed: int, n: int, count: int, t: int = 0):
    """Random (s, t) pairs with s != t (stream 7)."""
    s = np.array([uniform_int(seed, 7, t, 2 * q, 0, n - 1) for q in range(count)], np.int32)
    d = np.array([uniform_int(seed, 7, t, 2 * q + 1, 0, n - 2) for q in range(count)], np.int32)
    d = d + (d >= s)
    return s, d.astype(np.int32)
