"""Reference-side binding: tilefusion's numba kernels replaced by libtfb200.

This is the module a tilefusion maintainer would add to keep the reference
package itself (its Python API, pipeline, tests) and swap only the hot
kernels for the B200 ones.  ``install(tilefusion)``
rebinds the operator layer the reference's wrappers call through the
``_kernels`` module attribute (tsdf.py:127, :208, :269-279):

    _kernels.integrate_kernel(...)   (_kernels.py:71-88)   -> tf_integrate
    _kernels.raycast_kernel(...)     (_kernels.py:266-283) -> tf_raycast_ws
    _kernels.extract_bound(...)      (_kernels.py:454-478) -> tf_extract_count
    _kernels.extract_kernel(...)     (_kernels.py:481-578) -> tf_extract_emit

Same arguments, same in-place semantics on the caller's numpy arrays (each
call uploads the arrays, runs the kernel and writes the results back in
place, so it is slow by construction: the package ``paper_1511_07106_b200``
keeps volumes resident instead).  ``_sample`` (trilinear_sample's helper)
stays numba: it is a scalar host call.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from paper_1511_07106_b200 import _native as nat

CALLS = {"integrate_kernel": 0, "raycast_kernel": 0, "extract_bound": 0, "extract_kernel": 0}
_saved: dict = {}


def _vox(tsdf: np.ndarray, weight: np.ndarray) -> torch.Tensor:
    """(tsdf, weight) f32 [n][n][n] -> device float2 AoS (TfVolume layout)."""
    pair = np.stack([np.asarray(tsdf, np.float32), np.asarray(weight, np.float32)], -1)
    return torch.from_numpy(np.ascontiguousarray(pair)).to(nat.device())


def _volume(vox: torch.Tensor, n: int, ht, voxel_size: float) -> nat.TfVolume:
    return nat.volume_struct(vox, int(n), np.asarray(ht, np.int64), float(voxel_size))


def integrate_kernel(tsdf, weight, ht, voxel_size, depth, r_cw, t_cw, cam_center, fx, fy, cx, cy,
                     tau, max_weight, sample_weight):
    CALLS["integrate_kernel"] += 1
    n = tsdf.shape[0]
    vox = _vox(tsdf, weight)
    d = torch.from_numpy(np.ascontiguousarray(depth, np.float64)).to(nat.device())
    vol = _volume(vox, n, ht, voxel_size)
    cam = nat.TfCamera(float(fx), float(fy), float(cx), float(cy), depth.shape[1], depth.shape[0])
    L = nat.lib()
    ws = torch.empty(max(256, int(L.tf_integrate_workspace_size(ctypes.byref(vol), 1, ctypes.byref(cam)))),
                     dtype=torch.uint8, device=nat.device())
    nat.check(L.tf_integrate(ctypes.byref(vol), 1, nat.ptr(d), ctypes.byref(cam), nat.mat9(r_cw),
                             nat.vec3(t_cw), nat.vec3(cam_center), float(tau), float(max_weight),
                             float(sample_weight), nat.ptr(ws), ws.numel(), None, nat.stream_handle()),
              "tf_integrate")
    out = vox.cpu().numpy()
    tsdf[...] = out[..., 0]  # in place, like the numba kernel
    weight[...] = out[..., 1]


def raycast_kernel(tsdf, weight, ht, voxel_size, tau, coarse_step, r_wc, cam_center, fx, fy, cx, cy,
                   out_dist, out_vert, out_norm):
    CALLS["raycast_kernel"] += 1
    n = tsdf.shape[0]
    dev = nat.device()
    vox = _vox(tsdf, weight)
    vol = _volume(vox, n, ht, voxel_size)
    h, w = out_dist.shape
    cam = nat.TfCamera(float(fx), float(fy), float(cx), float(cy), w, h)
    dist = torch.from_numpy(np.ascontiguousarray(out_dist, np.float64)).to(dev)
    vert = torch.from_numpy(np.ascontiguousarray(out_vert, np.float64)).to(dev)
    norm = torch.from_numpy(np.ascontiguousarray(out_norm, np.float64)).to(dev)
    L = nat.lib()
    ws = torch.empty(int(L.tf_raycast_workspace_size(1, ctypes.byref(cam))), dtype=torch.uint8, device=dev)
    nat.check(L.tf_raycast_ws(ctypes.byref(vol), 1, ctypes.byref(cam), float(tau), int(coarse_step),
                              nat.mat9(r_wc), nat.vec3(cam_center), nat.ptr(dist), nat.ptr(vert),
                              nat.ptr(norm), nat.ptr(ws), ws.numel(), None, nat.stream_handle()),
              "tf_raycast_ws")
    out_dist[...] = dist.cpu().numpy()  # merged in place (_hit_wins), like the numba kernel
    out_vert[...] = vert.cpu().numpy()
    out_norm[...] = norm.cpu().numpy()


class _Extraction:
    """extract_bound's count is kept for the extract_kernel call that follows
    on the same arrays (tsdf.py:269-279 always calls them in that order)."""

    key = None
    count = 0


def extract_bound(tsdf, weight):
    CALLS["extract_bound"] += 1
    n = tsdf.shape[0]
    vox = _vox(tsdf, weight)
    vol = _volume(vox, n, np.zeros(3, np.int64), 1.0)
    L = nat.lib()
    ws = torch.empty(int(L.tf_extract_workspace_size(n)), dtype=torch.uint8, device=nat.device())
    cnt = torch.zeros(1, dtype=torch.int64, device=nat.device())
    nat.check(L.tf_extract_count(ctypes.byref(vol), nat.ptr(ws), ws.numel(), nat.ptr(cnt),
                                 nat.stream_handle()), "tf_extract_count")
    c = int(cnt.item())
    _Extraction.key, _Extraction.count = (id(tsdf), id(weight)), c
    return c


def extract_kernel(tsdf, weight, ht, voxel_size, out_verts, out_norms):
    CALLS["extract_kernel"] += 1
    n = tsdf.shape[0]
    vox = _vox(tsdf, weight)
    vol = _volume(vox, n, ht, voxel_size)
    L = nat.lib()
    dev = nat.device()
    ws = torch.empty(int(L.tf_extract_workspace_size(n)), dtype=torch.uint8, device=dev)
    cnt = torch.zeros(1, dtype=torch.int64, device=dev)
    nat.check(L.tf_extract_count(ctypes.byref(vol), nat.ptr(ws), ws.numel(), nat.ptr(cnt),
                                 nat.stream_handle()), "tf_extract_count")
    c = int(cnt.item())
    if c > out_verts.shape[0]:
        raise ValueError("extract_kernel: output smaller than extract_bound")
    verts = torch.empty((max(c, 1), 3), dtype=torch.float64, device=dev)
    norms = torch.empty((max(c, 1), 3), dtype=torch.float64, device=dev)
    if c:
        nat.check(L.tf_extract_emit(ctypes.byref(vol), nat.ptr(ws), ws.numel(), nat.ptr(verts),
                                    nat.ptr(norms), nat.stream_handle()), "tf_extract_emit")
        out_verts[:c] = verts[:c].cpu().numpy()
        out_norms[:c] = norms[:c].cpu().numpy()
    return c


_NAMES = ("integrate_kernel", "raycast_kernel", "extract_bound", "extract_kernel")


def install(tilefusion) -> None:
    """Rebind tilefusion._kernels' hot entry points to libtfb200."""
    k = tilefusion._kernels
    nat.load_library()
    for name in _NAMES:
        _saved.setdefault(name, getattr(k, name))
        setattr(k, name, globals()[name])


def uninstall(tilefusion) -> None:
    k = tilefusion._kernels
    for name, fn in _saved.items():
        setattr(k, name, fn)
    _saved.clear()
