"""Device-side inputs for the hot path: synthetic sphere volumes and APR
construction from pixels (generate_spheres, synthetic.hpp:74-111; build_apr,
build.hpp:290-312), through the C-ABI.  Used to make the C3/C4 workloads on the
GPU box in seconds (the reference builds 1024^3 in ~3 minutes and 34 GB RSS).
"""
from __future__ import annotations

import ctypes as C
from typing import Optional, Tuple

import numpy as np

from . import _lib as L
from .aprkit import APR, Context, DeviceApr, default_context


def generate_spheres(nz: int, nx: int, ny: int, count: int = 8, min_radius: float = 3.0, max_radius: float = 10.0,
                     background: float = 100.0, min_intensity: float = 500.0, max_intensity: float = 2000.0,
                     blur_sigma: float = 0.0, seed: int = 0, out_ptr: Optional[int] = None,
                     ctx: Optional[Context] = None) -> Optional[np.ndarray]:
    """generate_spheres (no noise).  Returns a host (nz,nx,ny) float32 array, or
    writes into the device buffer at out_ptr when given."""
    ctx = ctx or default_context()
    args = (ctx.handle, nz, nx, ny, count, float(min_radius), float(max_radius), float(background),
            float(min_intensity), float(max_intensity), float(blur_sigma), C.c_uint64(seed))
    if out_ptr is not None:
        L.check(L.lib().aprgpu_generate_spheres(*args, out_ptr, L.DEVICE))
        return None
    out = np.empty((nz, nx, ny), np.float32)
    L.check(L.lib().aprgpu_generate_spheres(*args, out.ctypes.data, L.HOST))
    return out


def _wrap_built(ctx: Context, h: C.c_void_p, dims) -> Tuple[APR, np.ndarray]:
    dev = DeviceApr(ctx, h, dims)
    apr = APR(dev.download(L.LEAF), dev.download(L.TREE), tuple(int(d) for d in dims))
    apr._dev[ctx.device] = dev
    vals = np.empty(dev.n_particles, np.float32)
    L.check(L.lib().aprgpu_apr_values(h, vals.ctypes.data, L.HOST))
    return apr, vals


def build_apr(volume, rel_error: float = 0.1, ctx: Optional[Context] = None) -> Tuple[APR, np.ndarray]:
    """build_apr with SigmaPolicy::constant(intensity_range(v)) on the GPU.
    volume: host (nz,nx,ny) float32 array, or a CUDA torch tensor."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    if hasattr(volume, "data_ptr"):
        nz, nx, ny = (int(s) for s in volume.shape)
        L.check(L.lib().aprgpu_build_apr(ctx.handle, volume.data_ptr(), nz, nx, ny, float(rel_error), L.DEVICE,
                                         C.byref(h)))
    else:
        v = np.ascontiguousarray(volume, np.float32)
        nz, nx, ny = v.shape
        L.check(L.lib().aprgpu_build_apr(ctx.handle, v.ctypes.data, nz, nx, ny, float(rel_error), L.HOST,
                                         C.byref(h)))
    return _wrap_built(ctx, h, (nz, nx, ny))


def build_apr_params(volume, params, ctx: Optional[Context] = None) -> Tuple[APR, np.ndarray]:
    """build_apr (build.hpp:290-312) with any BuildParams on the GPU: params is
    a paper_2112_03592_b200.BuildParams (sigma_mode 0 constant / 1 local range,
    gradient_mode 0 central difference / 1 Sobel, smoothing_passes).
    volume: host (nz,nx,ny) float32 array, or a CUDA torch tensor."""
    ctx = ctx or default_context()
    p = L.BuildParamsC(float(params.rel_error), int(params.sigma_mode), float(params.sigma_value),
                       int(params.sigma_window), float(params.sigma_floor), int(params.gradient_mode),
                       int(params.smoothing_passes))
    h = C.c_void_p()
    if hasattr(volume, "data_ptr"):
        nz, nx, ny = (int(s) for s in volume.shape)
        L.check(L.lib().aprgpu_build_apr_params(ctx.handle, volume.data_ptr(), nz, nx, ny, C.byref(p), L.DEVICE,
                                                C.byref(h)))
    else:
        v = np.ascontiguousarray(volume, np.float32)
        nz, nx, ny = v.shape
        L.check(L.lib().aprgpu_build_apr_params(ctx.handle, v.ctypes.data, nz, nx, ny, C.byref(p), L.HOST,
                                                C.byref(h)))
    return _wrap_built(ctx, h, (nz, nx, ny))


def build_spheres_apr(n, count: int, rmin: float, rmax: float, blur: float = 2.0, seed: int = 42,
                      rel_error: float = 0.1, ctx: Optional[Context] = None) -> Tuple[APR, np.ndarray]:
    """generate_spheres -> build_apr entirely on the device (the BASELINE.md
    configs: background 100, intensity U[500,2000], E = rel_error)."""
    import torch
    ctx = ctx or default_context()
    nz, nx, ny = (n, n, n) if np.isscalar(n) else tuple(n)
    vol = torch.empty((nz, nx, ny), dtype=torch.float32, device=f"cuda:{ctx.device}")
    generate_spheres(nz, nx, ny, count, rmin, rmax, 100.0, 500.0, 2000.0, blur, seed, out_ptr=vol.data_ptr(), ctx=ctx)
    torch.cuda.synchronize(ctx.device)
    try:
        return build_apr(vol, rel_error, ctx)
    finally:
        del vol
        torch.cuda.empty_cache()


def tile_apr(dev: DeviceApr, tz: int, tx: int, ty: int) -> DeviceApr:
    """The C4 tiler (aprgpu_tile_apr): a power-of-two cube APR on the device
    tiled (tz, tx, ty) times, structure and interior structure built on the
    device.  Returns the new device APR (no host copy: C4 is 548 M particles)."""
    h = C.c_void_p()
    L.check(L.lib().aprgpu_tile_apr(dev.handle, int(tz), int(tx), int(ty), C.byref(h)))
    dims = (dev.dims[0] * tz, dev.dims[1] * tx, dev.dims[2] * ty)
    return DeviceApr(dev.ctx, h, dims)


def tile_values(src: DeviceApr, big: DeviceApr, tz: int, tx: int, ty: int, src_ptr: int, big_ptr: int) -> None:
    """Particle values of `src` (device pointer) tiled like tile_apr into big_ptr."""
    L.check(L.lib().aprgpu_tile_values(src.handle, big.handle, int(tz), int(tx), int(ty), src_ptr, big_ptr))
