"""Torch-tensor binding of the optical-flow core (include/sgmflow.h, SURVEY.md
8(f) rank 2).  Marshalling only: every step runs in libsgmsf.so's kernels."""
from __future__ import annotations

import ctypes

import torch

from . import _lib
from .sgm import _ptr, _stream

FQ = 8   # flow vectors are integers in 1/FQ px


class FlowFields:
    """A libsgmsf optical-flow handle (pyramid, WHT/kNN init, propagation + random search,
    two inverse fields, consistency filter)."""

    def __init__(self, width, height, levels=3, patch_radius=4, sweeps=8, search_radius=8,
                 desc_window=8, knn=4, consistency_q=8, penalty=20, max_batch=1, seed=1,
                 device=0):
        self.lib = _lib.load()
        self.W, self.H = int(width), int(height)
        self.device = torch.device("cuda", device)
        self.params = _lib.SgmFlowParams(self.W, self.H, levels, patch_radius, sweeps,
                                         search_radius, desc_window, knn, consistency_q, penalty,
                                         max_batch, seed)
        self.knn = int(knn)
        self.radius = int(patch_radius)
        h = ctypes.c_void_p()
        _lib.call("sgm_flow_create", ctypes.byref(self.params), int(device), ctypes.byref(h))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.lib.sgm_flow_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    def launch_count(self) -> int:
        return int(self.lib.sgm_flow_launch_count(self.h))

    def set_timing(self, on: bool):
        _lib.call("sgm_flow_set_timing", self.h, 1 if on else 0)

    def read_timing(self):
        """{prop, search, knn} summed kernel ms of the last timed call, or None."""
        buf = (ctypes.c_float * 3)()
        if self.lib.sgm_flow_read_timing(self.h, buf) == 0:
            return None
        return {"prop": float(buf[0]), "search": float(buf[1]), "knn": float(buf[2])}

    def _empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device=self.device)

    def flow(self, frames0, frames1, want_fields=False, out=None, stream=None):
        """frames0 / frames1 uint8 [n][H][W] (device).  Returns dict flow float32
        [n][H][W][2] (px), valid uint8 [n][H][W] and, if asked, fields_q int32
        [n][3][H][W][2] (1/8 px)."""
        n = int(frames0.shape[0])
        if out is None:
            out = {"flow": self._empty((n, self.H, self.W, 2), torch.float32),
                   "valid": self._empty((n, self.H, self.W), torch.uint8)}
            if want_fields:
                out["fields_q"] = self._empty((n, 3, self.H, self.W, 2), torch.int32)
        _lib.call("sgm_flow", self.h, n, _ptr(frames0), _ptr(frames1), _ptr(out.get("flow")),
                  _ptr(out.get("valid")), _ptr(out.get("fields_q")), _stream(stream))
        return out

    def field(self, A, B, seed, radius=None, stream=None):
        n = int(A.shape[0])
        r = self.radius if radius is None else int(radius)
        f = self._empty((n, self.H, self.W, 2), torch.int32)
        c = self._empty((n, self.H, self.W), torch.int32)
        _lib.call("sgm_flow_field", self.h, n, _ptr(A), _ptr(B), int(seed), r, _ptr(f), _ptr(c),
                  _stream(stream))
        return f, c

    def descriptors(self, img, stream=None):
        h, w = img.shape
        d = self._empty((h, w, 16), torch.int32)
        _lib.call("sgm_flow_descriptors", self.h, _ptr(img), w, h, _ptr(d), _stream(stream))
        return d

    def patch_cost(self, A, B, queries, radius=None, stream=None):
        h, w = A.shape
        r = self.radius if radius is None else int(radius)
        q = queries.to(device=self.device, dtype=torch.int32).contiguous()
        out = self._empty((q.shape[0],), torch.int32)
        _lib.call("sgm_flow_patch_cost", self.h, _ptr(A), _ptr(B), w, h, r, int(q.shape[0]),
                  _ptr(q), _ptr(out), _stream(stream))
        return out

    def knn_init(self, A, B, radius=None, stream=None):
        h, w = A.shape
        r = self.radius if radius is None else int(radius)
        f = self._empty((h, w, 2), torch.int32)
        c = self._empty((h, w), torch.int32)
        nn = self._empty((h, w, self.knn), torch.int32)
        _lib.call("sgm_flow_knn_init", self.h, _ptr(A), _ptr(B), w, h, r, _ptr(f), _ptr(c), _ptr(nn),
                  _stream(stream))
        return f, c, nn

    def sweep(self, A, B, flow_q, cost, sweep, level=0, seed=1, radius=None, stream=None):
        """In place on flow_q / cost (device int32)."""
        h, w = A.shape
        r = self.radius if radius is None else int(radius)
        _lib.call("sgm_flow_sweep", self.h, _ptr(A), _ptr(B), w, h, r, int(sweep), int(level),
                  int(seed), _ptr(flow_q), _ptr(cost), _stream(stream))
        return flow_q, cost

    def consistency(self, F, G1, G2, stream=None):
        h, w = F.shape[:2]
        v = self._empty((h, w), torch.uint8)
        _lib.call("sgm_flow_consistency", self.h, _ptr(F), _ptr(G1), _ptr(G2), w, h, _ptr(v),
                  _stream(stream))
        return v


_densify_scratch = {}
# default candidate window of sgm_densify (Chebyshev px; 0 = every seed, the SPEC's F-6)
DENSIFY_WINDOW = 16


def densify(field, valid, guide, K=25, lam=1.0, window=DENSIFY_WINDOW, stream=None, count_unfilled=False,
            count_certified=False, scratch=None):
    """Edge-aware densification (sgm_densify, SPEC F-6): field float32 [n][H][W][C] (or
    [H][W][C]), valid / guide uint8 [n][H][W] (device).  window = 0: every seed competes
    (the SPEC's definition); > 0: seeds within Chebyshev max(window, rho_K).  Returns the
    dense field, plus the number of pixels of images without seeds and / or the number of
    gap pixels with a provably window-0 result if asked.  The scratch buffer is cached per
    shape and device unless one is passed."""
    squeeze = field.dim() == 3
    if squeeze:
        field, valid, guide = field[None], valid[None], guide[None]
    field = field.contiguous()
    n, H, W, C = field.shape
    out = torch.empty_like(field)
    cnt = torch.zeros((1,), dtype=torch.int32, device=field.device) if count_unfilled else None
    cert = torch.zeros((1,), dtype=torch.int32, device=field.device) if count_certified else None
    nbytes = int(_lib.load().sgm_densify_scratch_bytes(n, W, H))
    if scratch is None:
        key = (field.device, n, W, H)
        scratch = _densify_scratch.get(key)
        if scratch is None:
            scratch = torch.empty((nbytes,), dtype=torch.uint8, device=field.device)
            _densify_scratch[key] = scratch
    _lib.call("sgm_densify", n, W, H, C, _ptr(field), _ptr(valid.contiguous()), _ptr(guide.contiguous()),
              int(K), float(lam), int(window), _ptr(out), _ptr(cnt), _ptr(cert), _ptr(scratch), nbytes,
              _stream(stream))
    out = out[0] if squeeze else out
    res = (out,) + ((cnt,) if count_unfilled else ()) + ((cert,) if count_certified else ())
    return res[0] if len(res) == 1 else res
