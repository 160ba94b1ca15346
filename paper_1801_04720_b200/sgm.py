"""Python face of libsgmsf.so: the same entry points as include/sgmsf.h, taking torch
tensors.  PyTorch provides device memory and streams only; every step of the
method runs in the library's sm_100a kernels (argument marshalling only here).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass

import torch

from . import _lib

_U16 = getattr(torch, "uint16", torch.int16)
_U64 = getattr(torch, "uint64", torch.int64)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def pitch_for(width: int) -> int:
    """Row pitch (bytes) the TMA-staged census needs: a multiple of 16 >= width."""
    return (width + 15) // 16 * 16


@dataclass
class Camera:
    """Rectified pinhole rig (G19/G20)."""
    f_px: float
    baseline_m: float
    cx: float
    cy: float

    def c(self):
        return _lib.SgmCamera(self.f_px, self.baseline_m, self.cx, self.cy)


class SGM:
    """A libsgmsf handle: SGM stereo (census, cost, 8-path aggregation, WTA, LR) and
    the basic scene-flow combination on one device."""

    def __init__(self, width, height, num_disp, census_w=9, census_h=7, p1=7, p2=86,
                 lr_threshold=1, invalid_disp=-1, bilinear_rule=0, max_batch=1, device=0):
        self.lib = _lib.load()
        self.W, self.H, self.D = int(width), int(height), int(num_disp)
        self.device = torch.device("cuda", device)
        self.params = _lib.SgmParams(self.W, self.H, self.D, census_w, census_h, p1, p2,
                                     lr_threshold, invalid_disp, bilinear_rule, max_batch)
        h = ctypes.c_void_p()
        _lib.call("sgm_create", ctypes.byref(self.params), int(device), ctypes.byref(h))
        self.h = h
        self.max_batch = int(max_batch)
        self.pitch = pitch_for(self.W)

    @classmethod
    def from_config(cls, cfg, max_batch=1, device=0, bilinear_rule=0):
        return cls(cfg.W, cfg.H, cfg.D, cfg.cw, cfg.ch, cfg.P1, cfg.P2, cfg.T, -1, bilinear_rule,
                   max_batch, device)

    def close(self):
        if getattr(self, "h", None):
            self.lib.sgm_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover - best effort
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ geometry / info
    def geometry(self):
        v = [ctypes.c_int32() for _ in range(4)]
        _lib.call("sgm_get_geometry", self.h, *[ctypes.byref(x) for x in v])
        return {"Dp": v[0].value, "cells_per_lane": v[1].value, "sweep_warps": v[2].value,
                "band_rows": v[3].value}

    def launch_count(self) -> int:
        return int(self.lib.sgm_launch_count(self.h))

    def device_error(self, clear: bool = False) -> int:
        """Fault code of the handle's device fault word (0 = none); sgm_get_device_error.
        Call after synchronising the stream of the call in question."""
        code = ctypes.c_int32()
        _lib.call("sgm_get_device_error", self.h, ctypes.byref(code), 1 if clear else 0)
        return int(code.value)

    def set_debug_flags(self, flags: int):
        """sgm_debug_set_flags: 4 forces the sweeps' bounded waits to time out (tests)."""
        _lib.call("sgm_debug_set_flags", self.h, int(flags))

    def set_timing(self, on: bool):
        _lib.call("sgm_set_timing", self.h, 1 if on else 0)

    def read_timing(self):
        buf = (ctypes.c_float * _lib.NUM_STAGES)()
        n = self.lib.sgm_read_timing(self.h, buf)
        if n == 0:
            return None
        return {self.lib.sgm_stage_name(i).decode(): float(buf[i]) for i in range(n)}

    # ------------------------------------------------------------------ tensors
    def upload_image(self, img):
        """uint8 [H][W] (numpy or tensor) -> device tensor [H][pitch]."""
        t = torch.as_tensor(img, dtype=torch.uint8)
        out = torch.zeros((self.H, self.pitch), dtype=torch.uint8, device=self.device)
        out[:, : self.W].copy_(t)
        return out

    def _empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device=self.device)

    # ------------------------------------------------------------------ stage-wise ABI
    def census(self, img, out=None, stream=None):
        out = out if out is not None else self._empty((self.H, self.W), _U64)
        _lib.call("sgm_census", self.h, _ptr(img), int(img.stride(0)), _ptr(out), _stream(stream))
        return out

    def cost(self, cen_left, cen_right, view, out=None, stream=None):
        out = out if out is not None else self._empty((self.H, self.W, self.D), torch.uint8)
        _lib.call("sgm_cost", self.h, _ptr(cen_left), _ptr(cen_right), int(view), _ptr(out),
                  _stream(stream))
        return out

    def aggregate(self, cen_left, cen_right, view, out=None, stream=None):
        out = out if out is not None else self._empty((self.H, self.W, self.D), _U16)
        _lib.call("sgm_aggregate", self.h, _ptr(cen_left), _ptr(cen_right), int(view), _ptr(out),
                  _stream(stream))
        return out

    def wta(self, agg, stream=None):
        di = self._empty((self.H, self.W), torch.int16)
        ds = self._empty((self.H, self.W), torch.float32)
        _lib.call("sgm_wta", self.h, _ptr(agg), _ptr(di), _ptr(ds), _stream(stream))
        return di, ds

    def lr_check(self, dl_int, dl_sub, dr_int, stream=None):
        oi = self._empty((self.H, self.W), torch.int16)
        os_ = self._empty((self.H, self.W), torch.float32)
        v = self._empty((self.H, self.W), torch.uint8)
        _lib.call("sgm_lr_check", self.h, _ptr(dl_int), _ptr(dl_sub), _ptr(dr_int), _ptr(oi),
                  _ptr(os_), _ptr(v), _stream(stream))
        return oi, os_, v

    def disparity(self, left, right, stream=None):
        oi = self._empty((self.H, self.W), torch.int16)
        os_ = self._empty((self.H, self.W), torch.float32)
        v = self._empty((self.H, self.W), torch.uint8)
        assert left.stride(0) == right.stride(0)
        _lib.call("sgm_disparity", self.h, _ptr(left), _ptr(right), int(left.stride(0)), _ptr(oi),
                  _ptr(os_), _ptr(v), _stream(stream))
        return oi, os_, v

    def combine_sceneflow(self, d0, v0, d1, v1, flow, flow_valid=None, camera=None, with_3d=True,
                          stream=None):
        H, W = self.H, self.W
        sf = self._empty((H, W, 4), torch.float32)
        vsf = self._empty((H, W), torch.uint8)
        p0 = dp = v3 = None
        cam = None
        if with_3d:
            p0 = self._empty((H, W, 4), torch.float32)
            dp = self._empty((H, W, 4), torch.float32)
            v3 = self._empty((H, W), torch.uint8)
            cam = ctypes.byref(camera.c())
        _lib.call("sgm_combine_sceneflow", self.h, _ptr(d0), _ptr(v0), _ptr(d1), _ptr(v1),
                  _ptr(flow), _ptr(flow_valid), cam, _ptr(sf), _ptr(p0), _ptr(dp), _ptr(vsf),
                  _ptr(v3), _stream(stream))
        return {"sf": sf, "valid_sf": vsf, "p0": p0, "dp": dp, "valid_3d": v3}

    # ------------------------------------------------------------------ production path
    def alloc_outputs(self, n, with_3d=True, with_disp=True, pinned_host=False, with_p0=True,
                      stream_mode=False):
        """Output tensors for n quads.  stream_mode: disparities per frame, [n+1][H][W]."""
        H, W = self.H, self.W
        if pinned_host:
            mk = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=True)  # noqa: E731
        else:
            mk = lambda shape, dt: self._empty(shape, dt)  # noqa: E731
        out = {"sf": mk((n, H, W, 4), torch.float32), "valid_sf": mk((n, H, W), torch.uint8)}
        if with_3d:
            out.update(dp=mk((n, H, W, 4), torch.float32), valid_3d=mk((n, H, W), torch.uint8))
            if with_p0:
                out["p0"] = mk((n, H, W, 4), torch.float32)
        if with_disp:
            shp = (n + 1, H, W) if stream_mode else (n, 2, H, W)
            out.update(disp_int=mk(shp, torch.int16), disp_sub=mk(shp, torch.float32),
                       disp_valid=mk(shp, torch.uint8))
        return out

    @staticmethod
    def _out_struct(o):
        return _lib.SgmSceneflowOut(*[o[k].data_ptr() if o.get(k) is not None else None
                                      for k in ("sf", "valid_sf", "p0", "dp", "valid_3d",
                                                "disp_int", "disp_sub", "disp_valid")])

    def scene_flow(self, images, flow, camera, out=None, flow_valid=None, stream=None):
        """images: uint8 [n][4][H][pitch] device tensor (I_l^t, I_r^t, I_l^t+1, I_r^t+1);
        flow: float32 [n][H][W][2].  Returns the output dict (device tensors)."""
        n = int(images.shape[0])
        out = out if out is not None else self.alloc_outputs(n)
        o = self._out_struct(out)
        _lib.call("sgm_scene_flow", self.h, n, _ptr(images), int(images.stride(2)), _ptr(flow),
                  _ptr(flow_valid), ctypes.byref(camera.c()), ctypes.byref(o), _stream(stream))
        return out

    def scene_flow_stream(self, images, flow, camera, out=None, flow_valid=None, stream=None):
        """Streaming mode: images uint8 [n+1][2][H][pitch] device tensor (frame k =
        I_l^k, I_r^k of one video); flow float32 [n][H][W][2] (frame k -> k+1).  Quad k =
        (frame k, frame k+1); disparity outputs are per frame [n+1][H][W]."""
        n = int(flow.shape[0])
        if int(images.shape[0]) != n + 1:
            raise ValueError("stream mode needs n+1 frames for n flows")
        out = out if out is not None else self.alloc_outputs(n, stream_mode=True)
        o = self._out_struct(out)
        _lib.call("sgm_scene_flow_stream", self.h, n, _ptr(images), int(images.stride(2)),
                  _ptr(flow), _ptr(flow_valid), ctypes.byref(camera.c()), ctypes.byref(o),
                  _stream(stream))
        return out

    def scene_flow_stream_host(self, images, flow, camera, out, flow_valid=None, stream=None):
        """Host-buffer streaming mode: images uint8 [n+1][2][H][W], flow [n][H][W][2] and
        ``out`` (pinned) CPU tensors."""
        n = int(flow.shape[0])
        if int(images.shape[0]) != n + 1:
            raise ValueError("stream mode needs n+1 frames for n flows")
        o = self._out_struct(out)
        _lib.call("sgm_scene_flow_stream_host", self.h, n, _ptr(images), _ptr(flow),
                  _ptr(flow_valid), ctypes.byref(camera.c()), ctypes.byref(o), _stream(stream))
        return out

    def scene_flow_host(self, images, flow, camera, out, flow_valid=None, stream=None):
        """Host-buffer variant: images uint8 [n][4][H][W], flow float32 [n][H][W][2] and the
        tensors of ``out`` are (pinned) CPU tensors; copies run inside the call."""
        n = int(images.shape[0])
        o = self._out_struct(out)
        _lib.call("sgm_scene_flow_host", self.h, n, _ptr(images), _ptr(flow), _ptr(flow_valid),
                  ctypes.byref(camera.c()), ctypes.byref(o), _stream(stream))
        return out

    def evaluate(self, sf, valid_sf, gt_d0, gt_d1, gt_flow, gt_noc, gt_valid=None,
                 tau_abs=3.0, tau_rel=0.05, counts=None, stream=None):
        """KITTI outlier counts (sgm_evaluate): device tensors sf [n][H][W][4],
        valid_sf/gt_noc/gt_valid uint8 [n][H][W], gt_d0/gt_d1 float32 [n][H][W],
        gt_flow float32 [n][H][W][2].  Returns int64 counts [n][2][6] (device)."""
        n = int(sf.shape[0])
        if counts is None:
            counts = torch.empty((n, 2, 6), dtype=torch.int64, device=sf.device)
        _lib.call("sgm_evaluate", self.h, n, _ptr(sf), _ptr(valid_sf), _ptr(gt_d0), _ptr(gt_d1),
                  _ptr(gt_flow), _ptr(gt_valid), _ptr(gt_noc), float(tau_abs), float(tau_rel),
                  _ptr(counts), _stream(stream))
        return counts


def rates_from_counts(counts):
    """{split: {D1, D2, Fl, SF (percent of evaluated pixels), density (percent)}} from
    one [2][6] count block, computed by the library (sgm_eval_rates)."""
    c = (ctypes.c_uint64 * 12)(*[int(v) for row in counts for v in row])
    r = (ctypes.c_double * 10)()
    _lib.call("sgm_eval_rates", c, r)
    return {name: dict(zip(("D1", "D2", "Fl", "SF", "density"), r[5 * split:5 * split + 5]))
            for split, name in ((0, "occ"), (1, "noc"))}


def stack_video(video, pitch, device):
    """synth.make_video dict -> device frames [n+1][2][H][pitch], flow [n][H][W][2]."""
    left, right = video["left"], video["right"]
    nf, H, W = left.shape
    imgs = torch.zeros((nf, 2, H, pitch), dtype=torch.uint8)
    imgs[:, 0, :, :W] = torch.from_numpy(left)
    imgs[:, 1, :, :W] = torch.from_numpy(right)
    return imgs.to(device), torch.from_numpy(video["flow"]).to(device)


def stack_quads(quads, pitch, device):
    """Host quads (synth.make_quad dicts) -> device images [n][4][H][pitch], flow [n][H][W][2]."""
    n = len(quads)
    H, W = quads[0]["il0"].shape
    imgs = torch.zeros((n, 4, H, pitch), dtype=torch.uint8)
    flow = torch.empty((n, H, W, 2), dtype=torch.float32)
    for i, q in enumerate(quads):
        for k, key in enumerate(("il0", "ir0", "il1", "ir1")):
            imgs[i, k, :, :W] = torch.from_numpy(q[key])
        flow[i] = torch.from_numpy(q["flow"])
    return imgs.to(device), flow.to(device)
