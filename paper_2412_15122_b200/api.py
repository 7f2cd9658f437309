"""Torch-facing convenience wrapper over the C ABI (plumbing only).

PyTorch provides device memory (D, the workspace, edge vectors), the stream
and — for multi-GPU — the process group used to ship the 128-byte NCCL id.
Every step of the computation runs in libapsp_warm's CUDA kernels.
"""
from __future__ import annotations

import numpy as np
import torch

from . import _lib as L

_DT = {torch.int32: L.APSP_I32, torch.float32: L.APSP_F32}


class WarmAPSP:
    """Device-resident APSP matrix with warm-start updates (apsp_warm.h).

    W: (n, n) int32 or float32 tensor (any device; copied to ``device``), row-major
       W[i][j] = w(i -> j), diagonal 0, int32 absent edges = APSP_INF_I32.
    cap: capacity (max n over the handle's lifetime).
    """

    def __init__(self, W, directed=True, cap=None, device=None, stream=None, rank=0, world=1,
                 nccl_id=None, cold_start=True, semiring="shortest", local_group=None):
        W = torch.as_tensor(W)
        if W.dtype not in _DT:
            raise TypeError("W must be int32 or float32")
        n = W.shape[0]
        cap = n if cap is None else int(cap)
        self.device = torch.device(device if device is not None else
                                   (W.device if W.is_cuda else "cuda"))
        self.dtype = W.dtype
        self.cdtype = _DT[W.dtype]
        self.directed = bool(directed)
        self.cap, self.rank, self.world = cap, rank, world
        self.ld, self.row0, self.rows = L.apsp_layout(cap, world, rank)
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        with torch.cuda.device(self.device):
            self.D_local = torch.empty((max(self.rows, 1), self.ld), dtype=W.dtype, device=self.device)
            nbytes = L.apsp_workspace_bytes(self.cdtype, cap, world)
            self.workspace = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
            Wd = W.to(self.device).contiguous()
            # the copy ran on torch's current stream; the library reads W on its own
            self.stream.wait_stream(torch.cuda.current_stream(self.device))
            if local_group is not None:   # in-process rank group (apsp_create_local)
                self.h = L.apsp_create_local(self.cdtype, self.directed, n, cap, Wd.data_ptr(),
                                             Wd.stride(0), self.D_local.data_ptr(), self.ld,
                                             self.workspace.data_ptr(), nbytes, self.stream.cuda_stream,
                                             rank, local_group)
            else:
                self.h = L.apsp_create(self.cdtype, self.directed, n, cap, Wd.data_ptr(), Wd.stride(0),
                                       self.D_local.data_ptr(), self.ld, self.workspace.data_ptr(), nbytes,
                                       self.stream.cuda_stream, rank, world, nccl_id)
            del Wd
        if semiring not in ("shortest", "minimax"):
            raise ValueError("semiring must be 'shortest' or 'minimax'")
        self.semiring = semiring
        if semiring == "minimax":
            L.apsp_set_option(self.h, L.OPT_SEMIRING, 1)
        if cold_start:
            self.cold_fw()

    # ------------------------------------------------------------------ state
    @property
    def n(self) -> int:
        return L.apsp_size(self.h)

    @property
    def D(self) -> torch.Tensor:
        """This rank's rows of D (view), columns [0, n)."""
        n = self.n
        lo = min(self.row0, n)
        hi = min(self.row0 + self.rows, n)
        return self.D_local[: hi - lo, :n]

    def set_distances(self, Dfull):
        """Warm start from a known APSP matrix: copy this rank's rows."""
        n = self.n
        Dfull = torch.as_tensor(Dfull)
        lo, hi = min(self.row0, n), min(self.row0 + self.rows, n)
        self.D_local[: hi - lo, :n].copy_(Dfull[lo:hi, :n])
        self.sync_distances()

    def sync_distances(self):
        """D_local was written directly: let the library re-derive its image of it."""
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        L.apsp_sync_distances(self.h)

    @property
    def mirror_width(self):
        """Bits per entry of D's saturated copy the O(n^2) passes read (8, 16; 0: D itself)."""
        return L.apsp_mirror_width(self.h)

    def close(self):
        if getattr(self, "h", None):
            L.apsp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, opt, value):
        L.apsp_set_option(self.h, opt, value)

    def launches(self):
        return L.apsp_kernel_launches(self.h)

    # ------------------------------------------------------------------ operations
    def cold_fw(self):
        L.apsp_cold_fw(self.h)

    def add_node(self, out_w, in_w):
        out_w = self._vec(out_w)
        in_w = self._vec(in_w)
        x, info = L.apsp_add_node(self.h, out_w.data_ptr(), in_w.data_ptr())
        self._keep = (out_w, in_w)   # the stream may still read them
        return x, info

    def remove_node(self, k):
        return L.apsp_remove_node(self.h, int(k))

    def update_edge(self, u, v, w_new):
        return L.apsp_update_edge(self.h, int(u), int(v), float(w_new))

    def modify_edge_readd(self, u, v, w_new):
        """The paper's alg:APSPmodify: remove the cheaper endpoint,
        re-add it with the edited edge.  Returns (removed endpoint, info)."""
        return L.apsp_modify_edge_readd(self.h, int(u), int(v), float(w_new))

    def need_update_list(self, kind, a, b=-1, cap=None):
        """Test export: the affected pairs (rows, cols) a removal of node a
        (kind 'remove') or an increase of edge (a, b) (kind 'increase') would
        list, by the library's own detection kernels; nothing is applied."""
        k = {"remove": 4, "increase": 2}[kind]
        n = self.n
        cap = n * n if cap is None else int(cap)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        r, c, cnt = L.apsp_need_update_list(self.h, k, int(a), int(b), cap)
        return r, c, cnt

    def weight(self, u, v):
        """Current w(u -> v) as held on the device (WT)."""
        return L.apsp_get_weight(self.h, int(u), int(v), self.cdtype)

    def query(self, s, t, path_cap=4096):
        return L.sp_pair_query(self.h, int(s), int(t), self.cdtype, path_cap)

    def query_batch(self, s, t, path_cap=64):
        s = torch.as_tensor(s, dtype=torch.int32).to(self.device).contiguous()
        t = torch.as_tensor(t, dtype=torch.int32).to(self.device).contiguous()
        q = s.numel()
        dist = torch.empty(q, dtype=self.dtype, device=self.device)
        paths = torch.full((q, max(path_cap, 1)), -1, dtype=torch.int32, device=self.device)
        lens = torch.empty(q, dtype=torch.int32, device=self.device)
        nc = torch.empty(q, dtype=torch.int32, device=self.device)
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        L.sp_pair_query_batch(self.h, q, s.data_ptr(), t.data_ptr(), dist.data_ptr(), paths.data_ptr(),
                              path_cap, lens.data_ptr(), nc.data_ptr())
        return dist, paths, lens, nc

    def _vec(self, v):
        v = torch.as_tensor(v if not isinstance(v, np.ndarray) else np.ascontiguousarray(v))
        v = v.to(device=self.device, dtype=self.dtype).contiguous()
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        return v
