"""Host-side mirror of the reference's hot-path API (aprkit, C++ namespace
``aprkit``) over the B200 C-ABI.

Names, argument meaning and error behaviour follow the reference headers:

==========================  ==============================================
this module                 reference
==========================  ==============================================
LinearAccess                linear_access.hpp:52-96
APR, computational_ratio    apr.hpp:35-48
Stencil + presets           stencil.hpp:15-120
restrict_stencil            stencil.hpp:127-160
StencilPyramid/make_pyramid stencil.hpp:162-202
PadMode                     reconstruct.hpp:13
ConvolveOptions, RowSpan    convolve.hpp:20-29
nonempty_row_index          convolve.hpp:32-44
init_tree_structure         tree.hpp:26-82
fill_tree                   tree.hpp:110-150
convolve_apr                convolve.hpp:220-303
RLConfig, rl_apr            deconv.hpp:16-22, 75-107
==========================  ==============================================

Every compute call runs on the GPU through libaprgpu.so; there is no CPU path.
Host-array calls stage through device memory; ``DeviceApr`` exposes the
device-pointer (stream-ordered) entry points for callers that keep data in HBM.
"""
from __future__ import annotations

import ctypes as C
import enum
import os
import math
from dataclasses import dataclass, field
from typing import List, NamedTuple, Optional, Sequence, Tuple

import numpy as np

from . import _lib as L
from .errors import CapabilityError, IntegrityError, RangeError  # noqa: F401  (re-export)

kMaxYDim = 65536            # linear_access.hpp:17
kMaxStencilExtent = 13      # convolve.hpp:18


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


# ----------------------------------------------------------------- geometry --
def cell_size(l_max: int, l: int) -> int:               # linear_access.hpp:19
    return 1 << (l_max - l)


def grid_dim(pixel_dim: int, l_max: int, l: int) -> int:  # linear_access.hpp:21-24
    s = cell_size(l_max, l)
    return (pixel_dim + s - 1) // s


def compute_l_max(nz: int, nx: int, ny: int) -> int:     # linear_access.hpp:27-32
    m = max(nz, nx, ny)
    l = 0
    while (1 << l) < m:
        l += 1
    return l


def compute_l_min(l_max: int) -> int:                    # linear_access.hpp:34
    return min(1, l_max)


# -------------------------------------------------------------- structures --
class LinearAccess:
    """Per-level CSR sparse structure (linear_access.hpp:52-96)."""

    def __init__(self, l_min: int, l_max: int, z_dim, x_dim, y_dim, y_idx, xz_end, level_offset):
        self.l_min = int(l_min)
        self.l_max = int(l_max)
        self.z_dim = np.ascontiguousarray(z_dim, dtype=np.int32)
        self.x_dim = np.ascontiguousarray(x_dim, dtype=np.int32)
        self.y_dim = np.ascontiguousarray(y_dim, dtype=np.int32)
        self.y_idx = np.ascontiguousarray(y_idx, dtype=np.uint16)
        self.xz_end = np.ascontiguousarray(xz_end, dtype=np.uint64)
        self.level_offset = np.ascontiguousarray(level_offset, dtype=np.uint64)

    def particle_count(self) -> int:
        return int(self.y_idx.size)

    def row_count(self) -> int:
        return int(self.xz_end.size)

    def level_count(self) -> int:
        return self.l_max - self.l_min + 1

    def row_index(self, l: int, z: int, x: int) -> int:
        return int(self.level_offset[l]) + z * int(self.x_dim[l]) + x

    def get_row(self, l: int, z: int, x: int):
        if l < self.l_min or l > self.l_max:
            raise RangeError(f"get_row: level {l} outside [{self.l_min}, {self.l_max}]")
        if z < 0 or z >= self.z_dim[l] or x < 0 or x >= self.x_dim[l]:
            raise RangeError(f"get_row: (z, x) = ({z}, {x}) outside level {l} grid")
        r = self.row_index(l, z, x)
        b = 0 if r == 0 else int(self.xz_end[r - 1])
        return b, int(self.xz_end[r])

    def desc(self) -> L.AccessDesc:
        d = L.AccessDesc()
        d.l_min, d.l_max = self.l_min, self.l_max
        d.z_dim, d.x_dim, d.y_dim = _ptr(self.z_dim), _ptr(self.x_dim), _ptr(self.y_dim)
        d.y_idx = _ptr(self.y_idx) if self.y_idx.size else None
        d.n_particles = self.y_idx.size
        d.xz_end = _ptr(self.xz_end) if self.xz_end.size else None
        d.n_rows = self.xz_end.size
        d.level_offset = _ptr(self.level_offset)
        return d

    def equals(self, o: "LinearAccess") -> bool:
        return (self.l_min == o.l_min and self.l_max == o.l_max
                and all(np.array_equal(getattr(self, k)[self.l_min:], getattr(o, k)[o.l_min:])
                        for k in ("z_dim", "x_dim", "y_dim", "level_offset"))
                and np.array_equal(self.y_idx, o.y_idx) and np.array_equal(self.xz_end, o.xz_end))


@dataclass
class APR:
    """aprkit::APR (apr.hpp:35-44): leaf access, interior-node access, dims."""
    access: LinearAccess
    tree_access: Optional[LinearAccess]
    source_dims: Sequence[int]
    _dev: dict = field(default_factory=dict, repr=False, compare=False)

    def pixel_count(self) -> int:
        d = self.source_dims
        return int(d[0]) * int(d[1]) * int(d[2])

    def device(self, ctx: Optional["Context"] = None) -> "DeviceApr":
        """Upload (once per context) and return the device handle."""
        ctx = ctx or default_context()
        h = self._dev.get(ctx.device)
        if h is None:
            h = DeviceApr.upload(ctx, self)
            self._dev[ctx.device] = h
            if self.tree_access is None:
                self.tree_access = h.download(L.TREE)
        return h


@dataclass
class BuildParams:                                        # apr.hpp:16-33 (SigmaPolicy flattened)
    rel_error: float = 0.1
    sigma_mode: int = 0          # 0 constant, 1 local range
    sigma_value: float = 1.0
    sigma_window: int = 2
    sigma_floor: float = 0.0
    gradient_mode: int = 0       # 0 central difference, 1 Sobel
    smoothing_passes: int = 0


def load_apr(path: str, ctx: Optional["Context"] = None):
    """load_apr (io.hpp:178-183): (APR, leaf values).  The file is read straight
    into a device handle (validated on the device) and the host APR mirrors it;
    apr.params holds the stored BuildParams."""
    ctx = ctx or default_context()
    h = C.c_void_p()
    L.check(L.lib().aprgpu_load_apr(ctx.handle, os.fsencode(path), C.byref(h)))
    dims = np.zeros(3, np.int32)
    L.check(L.lib().aprgpu_apr_dims(h, _ptr(dims)))
    dev = DeviceApr(ctx, h, dims)
    apr = APR(dev.download(L.LEAF), dev.download(L.TREE), tuple(int(v) for v in dims))
    apr._dev[ctx.device] = dev
    values = np.empty(dev.n_particles, np.float32)
    if values.size:
        L.check(L.lib().aprgpu_apr_values(h, _ptr(values), L.HOST))
    p = L.BuildParamsC()
    L.check(L.lib().aprgpu_apr_params(h, C.byref(p)))
    apr.params = BuildParams(p.rel_error, p.sigma_mode, p.sigma_value, p.sigma_window, p.sigma_floor,
                             p.gradient_mode, p.smoothing_passes)
    return apr, values


def save_apr(path: str, apr: APR, values) -> None:
    """save_apr (io.hpp:171-176): byte-identical to the reference's writer."""
    values = np.ascontiguousarray(values, dtype=np.float32)
    if values.size != apr.access.particle_count():
        raise RangeError("write_apr: value count does not match particle count")
    dev = apr.device()
    L.check(L.lib().aprgpu_save_apr(dev.handle, os.fsencode(path), _ptr(values) if values.size else None, L.HOST))


@dataclass
class ValidationReport:                                   # apr.hpp:50-56
    ok: bool = True
    message: str = ""


def validate(apr_or_access, source_dims=None, ctx: Optional["Context"] = None) -> ValidationReport:
    """validate (apr.hpp:61-136) on the device in O(particles + rows): the
    reference's checks, order and messages without its O(pixels) cover map.
    Takes an APR, or a leaf LinearAccess and the image dims."""
    if isinstance(apr_or_access, APR):
        access, dims = apr_or_access.access, apr_or_access.source_dims
    else:
        access, dims = apr_or_access, source_dims
    ctx = ctx or default_context()
    d = access.desc()
    dm = np.array([int(v) for v in dims], np.int32)
    ok = C.c_int()
    buf = C.create_string_buffer(512)
    L.check(L.lib().aprgpu_validate_access(ctx.handle, C.byref(d), _ptr(dm), C.byref(ok), buf, 512))
    return ValidationReport(bool(ok.value), buf.value.decode())


def computational_ratio(apr: APR) -> float:              # apr.hpp:46-48
    return apr.pixel_count() / apr.access.particle_count()


class PadMode(enum.IntEnum):                              # reconstruct.hpp:13
    Zero = 0
    Reflect = 1


class PyramidMode(enum.IntEnum):                          # stencil.hpp:162
    Restricted = 0
    Rescaled = 1
    Uniform = 2
    Explicit = 3


@dataclass
class ConvolveOptions:                                    # convolve.hpp:20-23
    threads: int = 0            # accepted for API parity; the GPU path ignores it
    use_row_skip: bool = True   # accepted; results never depend on it
    accum: str = "exact"        # "exact": fp64, bit-identical to the reference; "fast": fp32


class RowSpan(NamedTuple):                                # convolve.hpp:26-29
    z: int
    x: int
    y_min: int
    y_max: int


# ----------------------------------------------------------------- stencils --
class Stencil:
    """Dense odd-extent stencil stored (z, x, y) row-major (stencil.hpp:15-44)."""

    def __init__(self, kz: int = 1, kx: int = 1, ky: int = 1, fill: float = 0.0, weights=None):
        if kz < 1 or kx < 1 or ky < 1 or kz % 2 == 0 or kx % 2 == 0 or ky % 2 == 0:
            raise RangeError("stencil extents must be odd and positive")
        self.kz, self.kx, self.ky = int(kz), int(kx), int(ky)
        if weights is None:
            self.weights = np.full(kz * kx * ky, fill, dtype=np.float32)
        else:
            self.weights = np.ascontiguousarray(weights, dtype=np.float32).reshape(-1).copy()
            if self.weights.size != kz * kx * ky:
                raise RangeError("stencil weight count does not match extents")

    def hz(self) -> int: return self.kz // 2
    def hx(self) -> int: return self.kx // 2
    def hy(self) -> int: return self.ky // 2

    def at(self, dz: int, dx: int, dy: int) -> float:
        return float(self.weights[((dz + self.hz()) * self.kx + (dx + self.hx())) * self.ky + (dy + self.hy())])

    def set(self, dz: int, dx: int, dy: int, v: float) -> None:
        self.weights[((dz + self.hz()) * self.kx + (dx + self.hx())) * self.ky + (dy + self.hy())] = v

    def sum(self) -> float:
        s = 0.0
        for w in self.weights.tolist():  # sequential double sum, stencil.hpp:39-43
            s += w
        return s

    def array(self) -> np.ndarray:
        return self.weights.reshape(self.kz, self.kx, self.ky)


def identity_stencil() -> Stencil:                        # stencil.hpp:46-50
    s = Stencil(1, 1, 1)
    s.weights[0] = 1.0
    return s


def box_stencil(k: int) -> Stencil:                       # stencil.hpp:52-55
    s = Stencil(k, k, k)
    L.check(L.lib().aprgpu_box_stencil(k, _ptr(s.weights)))
    return s


def gaussian_stencil(sigma: float, size: int = 0) -> Stencil:  # stencil.hpp:59-79
    k = C.c_int32(0)
    L.check(L.lib().aprgpu_gaussian_stencil(float(sigma), int(size), C.byref(k), None))
    s = Stencil(k.value, k.value, k.value)
    L.check(L.lib().aprgpu_gaussian_stencil(float(sigma), int(size), C.byref(k), _ptr(s.weights)))
    return s


def sobel_stencil(axis: int) -> Stencil:                  # stencil.hpp:83-98
    if axis < 0 or axis > 2:
        raise RangeError("sobel axis must be 0, 1 or 2")
    s = Stencil(3, 3, 3)
    L.check(L.lib().aprgpu_sobel_stencil(axis, _ptr(s.weights)))
    return s


def flip_stencil(w: Stencil) -> Stencil:                  # stencil.hpp:101-110
    return Stencil(w.kz, w.kx, w.ky, weights=w.array()[::-1, ::-1, ::-1])


def rescale_stencil(w: Stencil, delta: int) -> Stencil:   # stencil.hpp:114-120
    if delta < 0:
        raise RangeError("rescale_stencil: delta must be >= 0")
    return Stencil(w.kz, w.kx, w.ky, weights=w.weights * np.float32(math.ldexp(1.0, -delta)))


def restrict_stencil(w: Stencil, delta: int) -> Stencil:  # stencil.hpp:127-160
    k3 = (C.c_int32 * 3)()
    L.check(L.lib().aprgpu_restrict_stencil(_ptr(w.weights), w.kz, w.kx, w.ky, int(delta), k3, None))
    out = Stencil(k3[0], k3[1], k3[2])
    L.check(L.lib().aprgpu_restrict_stencil(_ptr(w.weights), w.kz, w.kx, w.ky, int(delta), k3,
                                            _ptr(out.weights)))
    return out


class StencilPyramid:
    """Per-level stencils for l in [l_min, l_max] (stencil.hpp:165-174)."""

    def __init__(self, l_min: int, l_max: int, mode: PyramidMode, stencils: List[Stencil]):
        self.l_min, self.l_max, self.mode, self.stencils = int(l_min), int(l_max), mode, stencils
        self._dev = {}

    def at(self, l: int) -> Stencil:
        if l < self.l_min or l > self.l_max:
            raise RangeError("StencilPyramid: level out of range")
        return self.stencils[l - self.l_min]

    def device(self, ctx: Optional["Context"] = None) -> "DevicePyramid":
        ctx = ctx or default_context()
        h = self._dev.get(ctx.device)
        if h is None:
            h = DevicePyramid(ctx, self)
            self._dev[ctx.device] = h
        return h


def make_pyramid(w: Stencil, l_min: int, l_max: int, mode: PyramidMode) -> StencilPyramid:  # stencil.hpp:176-191
    st = []
    for l in range(l_min, l_max + 1):
        delta = l_max - l
        if mode == PyramidMode.Restricted:
            st.append(restrict_stencil(w, delta))
        elif mode == PyramidMode.Rescaled:
            st.append(rescale_stencil(w, delta))
        else:
            st.append(Stencil(w.kz, w.kx, w.ky, weights=w.weights))
    return StencilPyramid(l_min, l_max, PyramidMode(mode), st)


def explicit_pyramid(stencils: List[Stencil], l_min: int, l_max: int) -> StencilPyramid:  # stencil.hpp:193-202
    if len(stencils) != l_max - l_min + 1:
        raise RangeError("explicit_pyramid: one stencil per level required")
    return StencilPyramid(l_min, l_max, PyramidMode.Explicit, list(stencils))


# ------------------------------------------------------------------ device --
class Context:
    """One aprgpu context (stream + launch counter) per GPU."""

    def __init__(self, device: int = 0):
        self.device = device
        h = C.c_void_p()
        L.check(L.lib().aprgpu_init(device, C.byref(h)))
        self.handle = h

    def stream(self) -> int:
        s = C.c_void_p()
        L.check(L.lib().aprgpu_ctx_stream(self.handle, C.byref(s)))
        return s.value or 0

    def launch_count(self) -> int:
        n = C.c_uint64()
        L.check(L.lib().aprgpu_launch_count(self.handle, C.byref(n)))
        return n.value


_CONTEXTS = {}


def default_context(device: int = 0) -> Context:
    ctx = _CONTEXTS.get(device)
    if ctx is None:
        ctx = Context(device)
        _CONTEXTS[device] = ctx
    return ctx


class DevicePyramid:
    def __init__(self, ctx: Context, pyr: StencilPyramid):
        self.ctx = ctx
        k3 = np.array([[s.kz, s.kx, s.ky] for s in pyr.stencils], dtype=np.int32).reshape(-1)
        w = np.concatenate([s.weights for s in pyr.stencils]).astype(np.float32)
        h = C.c_void_p()
        L.check(L.lib().aprgpu_pyramid_create_explicit(ctx.handle, _ptr(w), _ptr(k3), pyr.l_min, pyr.l_max,
                                                       C.byref(h)))
        self.handle = h
        self.l_min, self.l_max = pyr.l_min, pyr.l_max
        self.k3 = {pyr.l_min + i: (s.kz, s.kx, s.ky) for i, s in enumerate(pyr.stencils)}

    def half_width(self, l_lo: int, l_hi: int) -> int:
        """Largest stencil half-width over levels [l_lo, l_hi] (any axis)."""
        return max([max(k) // 2 for l, k in self.k3.items() if l_lo <= l <= l_hi] or [0])

    def __del__(self):
        try:
            if self.handle:
                L.lib().aprgpu_pyramid_free(self.handle)
        except Exception:
            pass


def _accum(opt_accum: str) -> int:
    if opt_accum == "exact":
        return L.ACCUM_EXACT
    if opt_accum == "fast":
        return L.ACCUM_FAST
    raise ValueError(f"unknown accumulation mode {opt_accum!r}")


class DeviceApr:
    """An APR uploaded to one GPU (leaf + interior structure, work lists)."""

    def __init__(self, ctx: Context, handle: C.c_void_p, dims):
        self.ctx, self.handle, self.dims = ctx, handle, tuple(int(d) for d in dims)
        self.n_particles = self.info(L.LEAF).n_particles
        self.n_tree = self.info(L.TREE).n_particles

    @classmethod
    def upload(cls, ctx: Context, apr: APR) -> "DeviceApr":
        dims = np.array(apr.source_dims, dtype=np.int32)
        ld = apr.access.desc()
        td = apr.tree_access.desc() if apr.tree_access is not None else None
        h = C.c_void_p()
        L.check(L.lib().aprgpu_upload_access(ctx.handle, C.byref(ld), C.byref(td) if td is not None else None,
                                              _ptr(dims), C.byref(h)))
        return cls(ctx, h, dims)

    def __del__(self):
        try:
            if self.handle:
                L.lib().aprgpu_apr_free(self.handle)
        except Exception:
            pass

    def info(self, which: int) -> L.AccessInfo:
        i = L.AccessInfo()
        L.check(L.lib().aprgpu_access_get_info(self.handle, which, C.byref(i)))
        return i

    def download(self, which: int, rows_only: bool = False) -> LinearAccess:
        """The access structure back in the reference layout; rows_only skips
        y_idx (the row geometry a slab plan needs, without C4's 1.1 GB)."""
        i = self.info(which)
        n = i.l_max + 1
        y = np.empty(0 if rows_only else i.n_particles, np.uint16)
        e = np.empty(i.n_rows, np.uint64)
        lo = np.zeros(n, np.uint64)
        zd, xd, yd = (np.zeros(n, np.int32) for _ in range(3))
        L.check(L.lib().aprgpu_download_access(self.handle, which, None if rows_only else _ptr(y), _ptr(e), _ptr(lo),
                                               _ptr(zd), _ptr(xd), _ptr(yd)))
        return LinearAccess(i.l_min, i.l_max, zd, xd, yd, y, e, lo)

    def row_index(self, level: int):
        cnt = C.c_uint64()
        L.check(L.lib().aprgpu_row_index(self.handle, level, None, None, None, None, 0, C.byref(cnt)))
        n = cnt.value
        z, x = np.empty(n, np.int32), np.empty(n, np.int32)
        y0, y1 = np.empty(n, np.uint16), np.empty(n, np.uint16)
        if n:
            L.check(L.lib().aprgpu_row_index(self.handle, level, _ptr(z), _ptr(x), _ptr(y0), _ptr(y1), n,
                                             C.byref(cnt)))
        return z, x, y0, y1

    # host-array entry points -------------------------------------------------
    def fill_tree(self, leaf: np.ndarray) -> np.ndarray:
        leaf = np.ascontiguousarray(leaf, dtype=np.float32)
        if leaf.size != self.n_particles:
            raise RangeError("fill_tree: leaf value count does not match the APR")
        out = np.empty(self.n_tree, np.float32)
        L.check(L.lib().aprgpu_fill_tree(self.handle, _ptr(leaf), _ptr(out) if out.size else None, L.HOST, None))
        return out

    def convolve(self, values: np.ndarray, tree: np.ndarray, pyr: DevicePyramid, pad: int, accum: int) -> np.ndarray:
        values = np.ascontiguousarray(values, dtype=np.float32)
        tree = np.ascontiguousarray(tree, dtype=np.float32)
        if values.size != self.n_particles or tree.size != self.n_tree:
            raise RangeError("convolve_apr: value counts do not match the APR")
        out = np.empty(self.n_particles, np.float32)
        L.check(L.lib().aprgpu_convolve(self.handle, _ptr(values), _ptr(tree) if tree.size else None, pyr.handle,
                                        int(pad), accum, _ptr(out), L.HOST, None))
        return out

    def rl(self, observed: np.ndarray, psf: Stencil, iterations: int, epsilon: float, accum: int,
           estimate=None) -> np.ndarray:
        """aprgpu_rl, or aprgpu_rl_resume from a running estimate (host arrays)."""
        observed = np.ascontiguousarray(observed, dtype=np.float32)
        out = np.empty(self.n_particles, np.float32)
        if estimate is None:
            L.check(L.lib().aprgpu_rl(self.handle, _ptr(observed), _ptr(psf.weights), psf.kz, psf.kx, psf.ky,
                                      int(iterations), float(epsilon), accum, _ptr(out), L.HOST, None))
        else:
            est = np.ascontiguousarray(estimate, dtype=np.float32)
            L.check(L.lib().aprgpu_rl_resume(self.handle, _ptr(observed), _ptr(est), _ptr(psf.weights), psf.kz,
                                             psf.kx, psf.ky, int(iterations), float(epsilon), accum, _ptr(out),
                                             L.HOST, None))
        return out

    def reconstruct_level(self, values: np.ndarray, tree_values, level: int) -> np.ndarray:
        values = np.ascontiguousarray(values, dtype=np.float32)
        if values.size != self.n_particles:
            raise RangeError("reconstruct_level: value count does not match the APR")
        tv = None
        if tree_values is not None and np.asarray(tree_values).size:
            tv = np.ascontiguousarray(tree_values, dtype=np.float32)
            if tv.size != self.n_tree:
                raise RangeError("reconstruct_level: tree value count does not match the APR")
        i = self.info(L.LEAF)
        if level < i.l_min or level > i.l_max:
            raise RangeError("reconstruct_level: level out of range")
        a = self.download_dims()
        nz, nx, ny = a[0][level], a[1][level], a[2][level]
        out = np.empty((nz, nx, ny), np.float32)
        L.check(L.lib().aprgpu_reconstruct_level(self.handle, _ptr(values), _ptr(tv) if tv is not None else None,
                                                 int(level), _ptr(out), L.HOST, None))
        return out

    def reconstruct_patch(self, values: np.ndarray, tree_values, spec: "PatchSpec") -> np.ndarray:
        values = np.ascontiguousarray(values, dtype=np.float32)
        tv = None
        if tree_values is not None and np.asarray(tree_values).size:
            tv = np.ascontiguousarray(tree_values, dtype=np.float32)
        c = L.PatchSpecC(spec.level, spec.z_begin, spec.z_end, spec.x_begin, spec.x_end, spec.pad, int(spec.pad_mode))
        i = self.info(L.LEAF)
        if spec.level < i.l_min or spec.level > i.l_max:
            raise RangeError("reconstruct_patch: level out of range")
        ny = self.download_dims()[2][spec.level]
        shape = (max(spec.z_end - spec.z_begin + 2 * spec.pad, 0), max(spec.x_end - spec.x_begin + 2 * spec.pad, 0),
                 ny + 2 * max(spec.pad, 0))
        out = np.empty(shape, np.float32)
        L.check(L.lib().aprgpu_reconstruct_patch(self.handle, _ptr(values), _ptr(tv) if tv is not None else None,
                                                 C.byref(c), _ptr(out) if out.size else None, L.HOST, None))
        return out

    def download_dims(self):
        """(z_dim, x_dim, y_dim) per level of the leaf access."""
        if not hasattr(self, "_dims_cache"):
            a = self.download(L.LEAF)
            self._dims_cache = (list(a.z_dim), list(a.x_dim), list(a.y_dim))
        return self._dims_cache

    # device-pointer entry points (stream-ordered; pointers are raw ints) -----
    def fill_tree_ptr(self, leaf_ptr: int, tree_ptr: int, stream: int = 0) -> None:
        L.check(L.lib().aprgpu_fill_tree(self.handle, leaf_ptr, tree_ptr, L.DEVICE, stream or None))

    def restrict(self, cut_level: int, z_lo: int, z_hi: int) -> None:
        """Per-tile state for the tiles meeting finest planes [z_lo, z_hi) at levels >= cut_level
        only (aprgpu_apr_restrict; before the first convolution)."""
        L.check(L.lib().aprgpu_apr_restrict(self.handle, int(cut_level), int(z_lo), int(z_hi)))

    def map_tiles(self) -> Tuple[int, int]:
        """(tile records held by the resident gather maps, output tiles of the APR)."""
        built, total = C.c_uint64(), C.c_uint64()
        L.check(L.lib().aprgpu_apr_map_tiles(self.handle, C.byref(built), C.byref(total)))
        return built.value, total.value

    def rebuild_index_ptr(self, stream: int = 0) -> None:
        """The paper protocol's per-call index step (aprgpu_rebuild_index)."""
        L.check(L.lib().aprgpu_rebuild_index(self.handle, stream or None))

    def convolve_ptr(self, values_ptr: int, tree_ptr: int, pyr: DevicePyramid, pad: int, accum: int, out_ptr: int,
                     stream: int = 0) -> None:
        L.check(L.lib().aprgpu_convolve(self.handle, values_ptr, tree_ptr, pyr.handle, int(pad), accum, out_ptr,
                                        L.DEVICE, stream or None))

    def reconstruct_level_ptr(self, values_ptr: int, tree_ptr: int, level: int, out_ptr: int,
                              stream: int = 0) -> None:
        L.check(L.lib().aprgpu_reconstruct_level(self.handle, values_ptr, tree_ptr or None, int(level), out_ptr,
                                                 L.DEVICE, stream or None))

    def rl_ptr(self, observed_ptr: int, psf: Stencil, iterations: int, epsilon: float, accum: int, out_ptr: int,
               stream: int = 0) -> None:
        L.check(L.lib().aprgpu_rl(self.handle, observed_ptr, _ptr(psf.weights), psf.kz, psf.kx, psf.ky,
                                  int(iterations), float(epsilon), accum, out_ptr, L.DEVICE, stream or None))


class MultiApr:
    """An APR cut into z-slabs over several devices in ONE process
    (aprgpu_multi_*: peer-to-peer halos, interior/boundary overlap; the C++
    drop-in's multi-GPU path).  devices may repeat (several slabs on one GPU)."""

    def __init__(self, apr: APR, devices: List[int], halo: int = 2):
        dims = np.array(apr.source_dims, dtype=np.int32)
        ld = apr.access.desc()
        td = apr.tree_access.desc() if apr.tree_access is not None else None
        devs = np.array(devices, dtype=np.int32)
        h = C.c_void_p()
        L.check(L.lib().aprgpu_multi_create(_ptr(devs), len(devices), C.byref(ld),
                                            C.byref(td) if td is not None else None, _ptr(dims), int(halo),
                                            C.byref(h)))
        self.handle = h
        self.n_particles = apr.access.particle_count()
        n, lc = C.c_int(), C.c_int()
        zb = np.zeros(2 * len(devices), np.int32)
        L.check(L.lib().aprgpu_multi_info(h, C.byref(n), C.byref(lc), _ptr(zb)))
        self.cut_level = lc.value
        self.bounds = [(int(zb[2 * i]), int(zb[2 * i + 1])) for i in range(n.value)]

    def convolve(self, values, tree_values, pyr: StencilPyramid, pad: PadMode = PadMode.Reflect,
                 accum: str = "exact") -> np.ndarray:
        v = np.ascontiguousarray(values, np.float32)
        tv = np.ascontiguousarray(tree_values, np.float32)
        k3 = np.array([[st.kz, st.kx, st.ky] for st in pyr.stencils], dtype=np.int32).reshape(-1)
        w = np.concatenate([st.weights for st in pyr.stencils]).astype(np.float32)
        out = np.empty(self.n_particles, np.float32)
        L.check(L.lib().aprgpu_multi_convolve(self.handle, _ptr(v), _ptr(tv) if tv.size else None, _ptr(w), _ptr(k3),
                                              pyr.l_min, pyr.l_max, int(pad), _accum(accum), _ptr(out)))
        return out

    def __del__(self):
        try:
            if self.handle:
                L.lib().aprgpu_multi_free(self.handle)
        except Exception:
            pass


# ----------------------------------------------------- reference front door --
def init_tree_structure(apr_access: LinearAccess, source_dims, ctx: Optional[Context] = None) -> LinearAccess:
    """tree.hpp:26-82 -- built on the GPU, bit-identical."""
    tmp = APR(apr_access, None, source_dims)
    h = DeviceApr.upload(ctx or default_context(), tmp)
    return h.download(L.TREE)


def nonempty_row_index(a: LinearAccess, source_dims=None, ctx: Optional[Context] = None) -> List[List[RowSpan]]:
    """convolve.hpp:32-44 -- computed on the GPU (per-level compaction)."""
    dims = source_dims if source_dims is not None else _dims_from_access(a)
    h = APR(a, None, dims).device(ctx)
    out = []
    for l in range(a.l_min, a.l_max + 1):
        z, x, y0, y1 = h.row_index(l)
        out.append([RowSpan(int(zz), int(xx), int(p), int(q)) for zz, xx, p, q in zip(z, x, y0, y1)])
    return out


def _dims_from_access(a: LinearAccess):
    return (int(a.z_dim[a.l_max]), int(a.x_dim[a.l_max]), int(a.y_dim[a.l_max]))


def fill_tree(apr: APR, leaf_values, threads: int = 0) -> np.ndarray:
    """tree.hpp:110-150 (threads accepted for parity; output never depends on it)."""
    return apr.device().fill_tree(leaf_values)


def convolve_apr(apr: APR, values, tree_values, pyramid: StencilPyramid, pad: PadMode = PadMode.Reflect,
                 opt: Optional[ConvolveOptions] = None) -> np.ndarray:
    """convolve.hpp:220-303."""
    opt = opt or ConvolveOptions()
    a = apr.access
    if pyramid.l_min > a.l_min or pyramid.l_max < a.l_max:
        raise RangeError("convolve_apr: pyramid does not cover the APR levels")
    for l in range(a.l_min, a.l_max + 1):
        w = pyramid.at(l)
        if w.kz > kMaxStencilExtent or w.kx > kMaxStencilExtent or w.ky > kMaxStencilExtent:
            raise CapabilityError("convolve_apr: stencil extent exceeds the supported maximum")
    dev = apr.device()
    return dev.convolve(values, tree_values, pyramid.device(dev.ctx), int(pad), _accum(opt.accum))


def convolve_pixels(v: np.ndarray, w: Stencil, pad: PadMode = PadMode.Reflect, threads: int = 0,
                    accum: str = "exact", ctx: Optional["Context"] = None) -> np.ndarray:
    """convolve.hpp:48-98 on the device: v is (nz, nx, ny) float32, y fastest.
    accum "exact" (default, bit-identical) or "fast" (fp32); threads is accepted
    for API parity."""
    del threads
    if w.kz > kMaxStencilExtent or w.kx > kMaxStencilExtent or w.ky > kMaxStencilExtent:
        raise CapabilityError("convolve_pixels: stencil extent exceeds the supported maximum")
    v = np.ascontiguousarray(v, dtype=np.float32)
    if v.ndim != 3:
        raise RangeError("convolve_pixels: expected a (nz, nx, ny) volume")
    ctx = ctx or default_context()
    out = np.empty_like(v)
    wt = np.ascontiguousarray(w.weights, dtype=np.float32)
    L.check(L.lib().aprgpu_convolve_pixels(ctx.handle, _ptr(v) if v.size else _ptr(wt), *v.shape, _ptr(wt), w.kz,
                                           w.kx, w.ky, int(pad), _accum(accum), _ptr(out) if v.size else _ptr(wt),
                                           L.HOST, None))
    return out


def convolve_pixels_ptr(ctx: "Context", in_ptr: int, dims, w: Stencil, pad: int, accum: int, out_ptr: int,
                        stream: int = 0) -> None:
    """Device-pointer convolve_pixels (stream-ordered)."""
    wt = np.ascontiguousarray(w.weights, dtype=np.float32)
    L.check(L.lib().aprgpu_convolve_pixels(ctx.handle, in_ptr, int(dims[0]), int(dims[1]), int(dims[2]), _ptr(wt),
                                           w.kz, w.kx, w.ky, int(pad), accum, out_ptr, L.DEVICE, stream or None))


@dataclass
class PatchSpec:                                          # reconstruct.hpp:28-35
    level: int = 0
    z_begin: int = 0
    z_end: int = 0
    x_begin: int = 0
    x_end: int = 0
    pad: int = 0
    pad_mode: PadMode = PadMode.Reflect


def reconstruct_level(apr: APR, values, tree_values, l: int) -> np.ndarray:
    """reconstruct.hpp:73-84 on the device: (z_dim, x_dim, y_dim) of level l."""
    if l < apr.access.l_min or l > apr.access.l_max:
        raise RangeError("reconstruct_level: level out of range")
    return apr.device().reconstruct_level(values, tree_values, l)


def reconstruct_full(apr: APR, values) -> np.ndarray:
    """reconstruct.hpp:87-90: every pixel takes its covering leaf's value."""
    return reconstruct_level(apr, values, None, apr.access.l_max)


def reconstruct_patch(apr: APR, values, tree_values, spec: PatchSpec) -> np.ndarray:
    """reconstruct.hpp:94-129 on the device."""
    return apr.device().reconstruct_patch(values, tree_values, spec)


@dataclass
class RLConfig:                                           # deconv.hpp:16-22
    iterations: int = 100
    psf: Stencil = field(default_factory=Stencil)
    epsilon: float = 0.0
    record_metrics_every: int = 0
    threads: int = 0
    accum: str = "exact"


def rl_apr(apr: APR, observed, cfg: RLConfig, observer=None) -> np.ndarray:
    """deconv.hpp:75-107, every iteration on the GPU.  With an observer the
    iterations run in blocks of record_metrics_every (the estimate is handed to
    the observer between blocks, as the reference does)."""
    dev = apr.device()
    acc = _accum(cfg.accum)
    if observer is None or cfg.record_metrics_every <= 0 or cfg.iterations <= 0:
        return dev.rl(observed, cfg.psf, cfg.iterations, cfg.epsilon, acc)
    # the reference's state between iterations is (u, eps, estimate): resuming
    # the device iteration every record_metrics_every iterations is bit-identical
    # to one uninterrupted run (aprgpu_rl_resume; deconv.hpp:103-104)
    every, done, est = cfg.record_metrics_every, 0, None
    while done < cfg.iterations:
        n = min(every, cfg.iterations - done)
        est = dev.rl(observed, cfg.psf, n, cfg.epsilon, acc, estimate=est)
        done += n
        if done % every == 0:
            observer(done, est)
    return est
