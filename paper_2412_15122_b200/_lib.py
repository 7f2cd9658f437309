"""ctypes binding of libapsp_warm.so (include/apsp_warm.h) — argument marshalling only.

Every function here has the same name and meaning as its C counterpart; all
computation happens in the library's CUDA kernels.  There is no fallback:
if the shared library is missing or fails to load, importing this module
raises.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libapsp_warm.so")

APSP_I32, APSP_F32 = 0, 1
APSP_INF_I32 = 0x3FFFFFFF
STATUS = {
    0: "APSP_OK", 1: "APSP_E_INVAL", 2: "APSP_E_RANGE", 3: "APSP_E_CAPACITY", 4: "APSP_E_PRECOND",
    5: "APSP_E_CUDA", 6: "APSP_E_NCCL", 7: "APSP_E_NOMEM", 8: "APSP_E_POISONED", 9: "APSP_E_UNSUPPORTED",
}
(OPT_FORCE_PATH, OPT_THETA, OPT_TAU, OPT_MAX_ROUNDS, OPT_ROW_DELTA, OPT_SEMIRING, OPT_FW16, OPT_MIRROR8,
 OPT_MIRROR, OPT_FUSED, OPT_HEAVY) = range(11)

# exported symbols (tests check the library exports every one of them)
SYMBOLS = [
    "apsp_layout", "apsp_workspace_bytes", "apsp_create", "apsp_destroy", "apsp_set_option",
    "apsp_cold_fw", "apsp_add_node", "apsp_remove_node", "apsp_update_edge", "sp_pair_query",
    "sp_pair_query_batch", "apsp_size", "apsp_last_error", "apsp_status_string",
    "apsp_nccl_unique_id", "apsp_kernel_launches", "apsp_profile_enable", "apsp_profile_reset",
    "apsp_profile_read", "apsp_modify_edge_readd", "apsp_get_weight",
    "apsp_local_group_create", "apsp_local_group_destroy", "apsp_create_local", "apsp_microbench",
    "apsp_sync_distances", "apsp_mirror_width", "apsp_need_update_list",
]
# kernel classes of apsp_profile_read (apsp_kernel_class)
K_CLASSES = ["fw_diag", "fw_panel", "fw_tile", "add_pass1", "rank1", "detect", "sparse0",
             "sparse_r", "query", "other", "emit"]


class UpdateInfo(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32), ("early_exit", ctypes.c_int32), ("path", ctypes.c_int32),
        ("rounds", ctypes.c_int32), ("affected_pairs", ctypes.c_int64),
        ("affected_rows", ctypes.c_int64), ("max_row_affected", ctypes.c_int64),
        ("cost", ctypes.c_double), ("n_after", ctypes.c_int64),
    ]

    def as_dict(self):
        return {f: getattr(self, f) for f, _ in self._fields_}


class ApspError(RuntimeError):
    def __init__(self, status, msg=""):
        self.status = status
        super().__init__(f"{STATUS.get(status, status)}: {msg}")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2412_15122_b200.build` "
            "(there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    i64, i32, vp, dbl = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p, ctypes.c_double
    P = ctypes.POINTER
    sig = {
        "apsp_layout": (ctypes.c_int, [i64, ctypes.c_int, ctypes.c_int, P(i64), P(i64), P(i64)]),
        "apsp_workspace_bytes": (ctypes.c_size_t, [ctypes.c_int, i64, ctypes.c_int]),
        "apsp_create": (ctypes.c_int, [P(vp), ctypes.c_int, ctypes.c_int, i64, i64, vp, i64, vp, i64, vp,
                                       ctypes.c_size_t, vp, ctypes.c_int, ctypes.c_int, vp]),
        "apsp_local_group_create": (ctypes.c_int, [ctypes.c_int, P(vp)]),
        "apsp_local_group_destroy": (ctypes.c_int, [vp]),
        "apsp_create_local": (ctypes.c_int, [P(vp), ctypes.c_int, ctypes.c_int, i64, i64, vp, i64, vp, i64,
                                             vp, ctypes.c_size_t, vp, ctypes.c_int, vp]),
        "apsp_microbench": (ctypes.c_int, [ctypes.c_int, vp, ctypes.c_size_t, vp, P(dbl)]),
        "apsp_destroy": (ctypes.c_int, [vp]),
        "apsp_set_option": (ctypes.c_int, [vp, ctypes.c_int, dbl]),
        "apsp_cold_fw": (ctypes.c_int, [vp]),
        "apsp_sync_distances": (ctypes.c_int, [vp]),
        "apsp_mirror_width": (ctypes.c_int32, [vp]),
        "apsp_add_node": (ctypes.c_int, [vp, vp, vp, P(i64), P(UpdateInfo)]),
        "apsp_remove_node": (ctypes.c_int, [vp, i64, P(i64), P(UpdateInfo)]),
        "apsp_update_edge": (ctypes.c_int, [vp, i64, i64, dbl, P(UpdateInfo)]),
        "apsp_modify_edge_readd": (ctypes.c_int, [vp, i64, i64, dbl, P(i64), P(UpdateInfo)]),
        "sp_pair_query": (ctypes.c_int, [vp, i64, i64, vp, P(i32), i32, P(i32), P(i32)]),
        "sp_pair_query_batch": (ctypes.c_int, [vp, i32, vp, vp, vp, vp, i32, vp, vp]),
        "apsp_size": (i64, [vp]),
        "apsp_get_weight": (ctypes.c_int, [vp, i64, i64, vp]),
        "apsp_need_update_list": (ctypes.c_int, [vp, i32, i64, i64, vp, vp, i64, P(i64)]),
        "apsp_last_error": (ctypes.c_char_p, [vp]),
        "apsp_status_string": (ctypes.c_char_p, [ctypes.c_int]),
        "apsp_nccl_unique_id": (ctypes.c_int, [vp]),
        "apsp_kernel_launches": (i64, [vp]),
        "apsp_profile_enable": (ctypes.c_int, [vp, ctypes.c_int]),
        "apsp_profile_reset": (ctypes.c_int, [vp]),
        "apsp_profile_read": (ctypes.c_int, [vp, ctypes.c_int, P(dbl), P(i64), P(dbl)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    return L


lib = _load()


def check(h, status):
    if status != 0:
        msg = lib.apsp_last_error(h).decode() if h else lib.apsp_status_string(status).decode()
        raise ApspError(status, msg)


# ---------------------------------------------------------------- same-name wrappers
def apsp_layout(cap, world=1, rank=0):
    ld, row0, rows = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    check(None, lib.apsp_layout(cap, world, rank, ctypes.byref(ld), ctypes.byref(row0), ctypes.byref(rows)))
    return ld.value, row0.value, rows.value


def apsp_workspace_bytes(dtype, cap, world=1):
    return int(lib.apsp_workspace_bytes(dtype, cap, world))


def apsp_create(dtype, directed, n, cap, W_ptr, ldw, D_ptr, ld, ws_ptr, ws_bytes, stream, rank=0,
                world=1, nccl_id=None):
    h = ctypes.c_void_p()
    idbuf = None
    if nccl_id is not None:
        idbuf = ctypes.create_string_buffer(bytes(nccl_id), 128)
    st = lib.apsp_create(ctypes.byref(h), dtype, int(directed), n, cap, W_ptr, ldw, D_ptr, ld, ws_ptr,
                         ws_bytes, stream, rank, world, idbuf)
    check(None, st)
    return h


def apsp_local_group_create(world):
    g = ctypes.c_void_p()
    check(None, lib.apsp_local_group_create(world, ctypes.byref(g)))
    return g


def apsp_local_group_destroy(g):
    check(None, lib.apsp_local_group_destroy(g))


def apsp_create_local(dtype, directed, n, cap, W_ptr, ldw, D_ptr, ld, ws_ptr, ws_bytes, stream, rank,
                      group):
    h = ctypes.c_void_p()
    check(None, lib.apsp_create_local(ctypes.byref(h), dtype, int(directed), n, cap, W_ptr, ldw, D_ptr, ld,
                                      ws_ptr, ws_bytes, stream, rank, group))
    return h


def apsp_microbench(kind, buf_ptr, nbytes, stream):
    """K13 roofline denominators (apsp_warm.h): 0 int32 / 1 fp32 / 2 int16x2
    relaxations per second, 3 HBM read / 4 read+write bytes per second."""
    r = ctypes.c_double()
    check(None, lib.apsp_microbench(kind, buf_ptr, nbytes, stream, ctypes.byref(r)))
    return r.value


def apsp_destroy(h):
    check(None, lib.apsp_destroy(h))


def apsp_set_option(h, opt, value):
    check(h, lib.apsp_set_option(h, opt, float(value)))


def apsp_sync_distances(h):
    check(h, lib.apsp_sync_distances(h))


def apsp_mirror_width(h):
    return int(lib.apsp_mirror_width(h))


def apsp_cold_fw(h):
    check(h, lib.apsp_cold_fw(h))


def apsp_add_node(h, out_ptr, in_ptr):
    x = ctypes.c_int64()
    info = UpdateInfo()
    check(h, lib.apsp_add_node(h, out_ptr, in_ptr, ctypes.byref(x), ctypes.byref(info)))
    return x.value, info


def apsp_remove_node(h, k):
    mf = ctypes.c_int64()
    info = UpdateInfo()
    check(h, lib.apsp_remove_node(h, k, ctypes.byref(mf), ctypes.byref(info)))
    return mf.value, info


def apsp_update_edge(h, u, v, w_new):
    info = UpdateInfo()
    check(h, lib.apsp_update_edge(h, u, v, float(w_new), ctypes.byref(info)))
    return info


def apsp_modify_edge_readd(h, u, v, w_new):
    removed = ctypes.c_int64(-1)
    info = UpdateInfo()
    check(h, lib.apsp_modify_edge_readd(h, u, v, float(w_new), ctypes.byref(removed), ctypes.byref(info)))
    return removed.value, info


def sp_pair_query(h, s, t, dtype, path_cap=4096):
    dist = ctypes.c_int32() if dtype == APSP_I32 else ctypes.c_float()
    path = (ctypes.c_int32 * max(path_cap, 1))()
    plen, nc = ctypes.c_int32(), ctypes.c_int32()
    check(h, lib.sp_pair_query(h, s, t, ctypes.byref(dist), path, path_cap, ctypes.byref(plen),
                               ctypes.byref(nc)))
    return dist.value, list(path[: plen.value]), nc.value


def sp_pair_query_batch(h, q, s_ptr, t_ptr, dist_ptr, paths_ptr, path_cap, lens_ptr, ncand_ptr):
    check(h, lib.sp_pair_query_batch(h, q, s_ptr, t_ptr, dist_ptr, paths_ptr, path_cap, lens_ptr, ncand_ptr))


def apsp_get_weight(h, u, v, dtype):
    w = ctypes.c_int32() if dtype == APSP_I32 else ctypes.c_float()
    check(h, lib.apsp_get_weight(h, u, v, ctypes.byref(w)))
    return w.value


def apsp_need_update_list(h, kind, a, b, cap):
    """(rows, cols, |A|) of a prospective removal (kind 4, node a) or edge
    increase (kind 2, edge (a, b)); test / diagnostic export (apsp_warm.h)."""
    import numpy as np

    rows = np.empty(max(cap, 1), np.int32)
    cols = np.empty(max(cap, 1), np.int32)
    cnt = ctypes.c_int64()
    check(h, lib.apsp_need_update_list(h, kind, a, b, rows.ctypes.data, cols.ctypes.data, cap,
                                       ctypes.byref(cnt)))
    m = min(cnt.value, cap)
    return rows[:m], cols[:m], cnt.value


def apsp_size(h):
    return int(lib.apsp_size(h))


def apsp_kernel_launches(h):
    return int(lib.apsp_kernel_launches(h))


def apsp_nccl_unique_id():
    buf = ctypes.create_string_buffer(128)
    check(None, lib.apsp_nccl_unique_id(buf))
    return buf.raw


def apsp_profile_enable(h, on=True):
    check(h, lib.apsp_profile_enable(h, int(on)))


def apsp_profile_reset(h):
    check(h, lib.apsp_profile_reset(h))


def apsp_profile_read(h):
    """{class: (ms, launches, algorithmic work)} accumulated since the last reset."""
    out = {}
    for c, name in enumerate(K_CLASSES):
        ms, cnt, work = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
        check(h, lib.apsp_profile_read(h, c, ctypes.byref(ms), ctypes.byref(cnt), ctypes.byref(work)))
        out[name] = (ms.value, cnt.value, work.value)
    return out
