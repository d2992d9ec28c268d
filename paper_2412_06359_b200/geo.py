"""The geometry-consistency loss L_geo on the device,
mirroring the reference's names and semantics (geometry.hpp:329-543):

  GeoLossTerms, geometry_consistency_loss             geometry.hpp:329-336, 416-453
  GeoLossGrad, geometry_consistency_loss_backward     geometry.hpp:338-344, 458-534
  total_loss, GEO_WEIGHT_DEFAULT                      geometry.hpp:538-543

plus ``geometry_consistency_loss_batch``, which evaluates one depth pair under
many poses in one call (how predictor_loss_and_gradients uses it, one pose per
bin, optimize.hpp:219-236). Everything runs through libevcm_cuda.so
(evcm_cuda_geometry_consistency_loss, csrc/geo.cu); there is no CPU fallback.
Depth maps are [H, W] float64 numpy arrays or torch CUDA tensors; masks are
optional uint8 [H, W] (nonzero = valid, DepthMap::valid, types.hpp:323-339).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from .engine import (MEM_DEVICE, DimensionMismatchError, Engine, _is_torch, _k_array, _mem_of,
                     _ptr, _raise, default_engine, load_library)

GEO_WEIGHT_DEFAULT = 0.05  # kGeoWeightDefault (geometry.hpp:538)


class _GeoOut(C.Structure):
    _fields_ = [("value", C.c_void_p), ("n_valid", C.c_void_p), ("projected", C.c_void_p),
                ("interpolated", C.c_void_p), ("valid", C.c_void_p), ("d_d0", C.c_void_p),
                ("d_d1", C.c_void_p), ("d_poses", C.c_void_p), ("d_depth_sum", C.c_void_p)]


@dataclass
class GeoLossTerms:
    """GeoLossTerms (geometry.hpp:329-336)."""
    projected: object
    interpolated: object
    valid: object
    value: float = 0.0
    n_valid: int = 0
    empty_valid_set: bool = True


@dataclass
class GeoLossGrad:
    """GeoLossGrad (geometry.hpp:338-344): d_omega / d_trans as length-3 arrays."""
    terms: GeoLossTerms
    d_d0: object
    d_d1: object
    d_omega: object
    d_trans: object


@dataclass
class GeoBatch:
    """One depth pair under n poses: per-pose value / n_valid [n], terms and
    gradients [n, H, W], d_poses [n, 6] and the summed depth gradient [H, W]."""
    value: object
    n_valid: object
    projected: object
    interpolated: object
    valid: object
    d_d0: object = None
    d_d1: object = None
    d_poses: object = None
    d_depth_sum: object = None


def _alloc(dev, shape, dtype):
    if dev is not None:
        import torch
        t = {np.float64: torch.float64, np.int64: torch.int64, np.uint8: torch.uint8}[dtype]
        return torch.zeros(shape, dtype=t, device=dev)
    return np.zeros(shape, dtype)


def geometry_consistency_loss_batch(d0, d1, poses, k, mask0=None, mask1=None,
                                    upstream: float = 1.0, want_grad: bool = True,
                                    engine: Optional[Engine] = None) -> GeoBatch:
    """geometry_consistency_loss[_backward] of d0 -> d1 for each pose row
    {omega xyz, trans xyz} of ``poses`` [n, 6]."""
    e = engine or default_engine()
    if tuple(d0.shape) != tuple(d1.shape) or len(d0.shape) != 2:
        raise DimensionMismatchError("depth consistency: depth maps must share a shape")
    for m in (mask0, mask1):
        if m is not None and tuple(m.shape) != tuple(d0.shape):
            raise DimensionMismatchError("depth map: mask shape must match depth shape")
    mem = _mem_of(d0, d1, poses, mask0, mask1)
    H, W = d0.shape
    if mem == MEM_DEVICE:
        dev = d0.device
    else:
        dev = None
        d0 = np.ascontiguousarray(d0, np.float64)
        d1 = np.ascontiguousarray(d1, np.float64)
        mask0 = None if mask0 is None else np.ascontiguousarray(mask0, np.uint8)
        mask1 = None if mask1 is None else np.ascontiguousarray(mask1, np.uint8)
        poses = np.ascontiguousarray(poses, np.float64)
    poses = poses.reshape(-1, 6)
    n = int(poses.shape[0])
    out = GeoBatch(_alloc(dev, (n,), np.float64), _alloc(dev, (n,), np.int64),
                   _alloc(dev, (n, H, W), np.float64), _alloc(dev, (n, H, W), np.float64),
                   _alloc(dev, (n, H, W), np.uint8))
    if want_grad:
        out.d_d0 = _alloc(dev, (n, H, W), np.float64)
        out.d_d1 = _alloc(dev, (n, H, W), np.float64)
        out.d_poses = _alloc(dev, (n, 6), np.float64)
        out.d_depth_sum = _alloc(dev, (H, W), np.float64)
    go = _GeoOut(_ptr(out.value), _ptr(out.n_valid), _ptr(out.projected), _ptr(out.interpolated),
                 _ptr(out.valid), _ptr(out.d_d0), _ptr(out.d_d1), _ptr(out.d_poses),
                 _ptr(out.d_depth_sum))
    e._order_after(d0, d1, poses)
    _raise(load_library().evcm_cuda_geometry_consistency_loss(
        e._h, W, H, _ptr(d0), _ptr(mask0), _ptr(d1), _ptr(mask1), n, _ptr(poses),
        _ptr(_k_array(k)), float(upstream), int(want_grad), mem, C.byref(go)))
    return out


def _terms(b: GeoBatch) -> GeoLossTerms:
    nv = int(b.n_valid[0])
    return GeoLossTerms(b.projected[0], b.interpolated[0], b.valid[0], float(b.value[0]), nv,
                        nv == 0)


def geometry_consistency_loss(d0, d1, pose, k, mask0=None, mask1=None,
                              engine: Optional[Engine] = None) -> GeoLossTerms:
    """geometry_consistency_loss (geometry.hpp:416-453): mean |a - b| / (a + b)
    over the valid set of the z-min forward projection of d0 into d1."""
    return _terms(geometry_consistency_loss_batch(d0, d1, pose, k, mask0, mask1, 1.0, False,
                                                  engine))


def geometry_consistency_loss_backward(d0, d1, pose, k, upstream: float = 1.0, mask0=None,
                                       mask1=None, engine: Optional[Engine] = None) -> GeoLossGrad:
    """geometry_consistency_loss_backward (geometry.hpp:458-534): the loss plus
    its gradients w.r.t. both depth maps and the pose, scaled by ``upstream``."""
    b = geometry_consistency_loss_batch(d0, d1, pose, k, mask0, mask1, upstream, True, engine)
    return GeoLossGrad(_terms(b), b.d_d0[0], b.d_d1[0], b.d_poses[0, :3], b.d_poses[0, 3:])


def total_loss(contrast: float, geo: float, weight: float = GEO_WEIGHT_DEFAULT) -> float:
    """total_loss (geometry.hpp:540-543)."""
    return contrast + weight * geo
