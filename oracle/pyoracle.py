"""oracle/pyoracle.py -- TEST INFRASTRUCTURE ONLY.

ctypes bindings of
  * oracle/liboracle.so      -- the plain-C restatement (aprk_oracle.c), and
  * oracle/_ref/libaprref.so -- the unmodified reference compiled where it lies
                               (ref_shim.cpp), when it has been built.
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import
this module, and only as the checker / the timed CPU baseline.

Access structures are exchanged as ``Access`` objects whose attribute names
match the product's ``LinearAccess`` (duck-typed both ways).
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libaprref.so")


@dataclass
class Access:
    l_min: int
    l_max: int
    z_dim: np.ndarray
    x_dim: np.ndarray
    y_dim: np.ndarray
    y_idx: np.ndarray
    xz_end: np.ndarray
    level_offset: np.ndarray

    def particle_count(self):
        return int(self.y_idx.size)


def as_access(a) -> Access:
    return Access(int(a.l_min), int(a.l_max), np.ascontiguousarray(a.z_dim, np.int32),
                  np.ascontiguousarray(a.x_dim, np.int32), np.ascontiguousarray(a.y_dim, np.int32),
                  np.ascontiguousarray(a.y_idx, np.uint16), np.ascontiguousarray(a.xz_end, np.uint64),
                  np.ascontiguousarray(a.level_offset, np.uint64))


def _p(a: np.ndarray):
    return a.ctypes.data if a.size else None


# ------------------------------------------------------------- C oracle ----
class _OrcAccess(C.Structure):
    _fields_ = [("l_min", C.c_int), ("l_max", C.c_int), ("z_dim", C.c_void_p), ("x_dim", C.c_void_p),
                ("y_dim", C.c_void_p), ("y_idx", C.c_void_p), ("n_particles", C.c_uint64),
                ("xz_end", C.c_void_p), ("n_rows", C.c_uint64), ("level_offset", C.c_void_p)]


class _OrcOwned(C.Structure):
    _fields_ = [("l_min", C.c_int), ("l_max", C.c_int), ("z_dim", C.POINTER(C.c_int)),
                ("x_dim", C.POINTER(C.c_int)), ("y_dim", C.POINTER(C.c_int)), ("y_idx", C.POINTER(C.c_uint16)),
                ("n_particles", C.c_uint64), ("xz_end", C.POINTER(C.c_uint64)), ("n_rows", C.c_uint64),
                ("level_offset", C.POINTER(C.c_uint64))]


class _OrcPyr(C.Structure):
    _fields_ = [("l_min", C.c_int), ("l_max", C.c_int), ("k3", C.c_void_p), ("w", C.c_void_p), ("off", C.c_void_p)]


def _orc_access(a: Access, keep: list) -> _OrcAccess:
    a = as_access(a)
    keep.append(a)
    s = _OrcAccess()
    s.l_min, s.l_max = a.l_min, a.l_max
    s.z_dim, s.x_dim, s.y_dim = a.z_dim.ctypes.data, a.x_dim.ctypes.data, a.y_dim.ctypes.data
    s.y_idx, s.n_particles = _p(a.y_idx), a.y_idx.size
    s.xz_end, s.n_rows = _p(a.xz_end), a.xz_end.size
    s.level_offset = a.level_offset.ctypes.data
    return s


class Oracle:
    """The plain-C restatement."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            raise RuntimeError(f"oracle not built: {path} (run `make oracle`)")
        self.L = C.CDLL(path)
        vp = C.c_void_p
        L = self.L
        L.orc_reflect_index.restype = C.c_int
        L.orc_reflect_index.argtypes = [C.c_int, C.c_int]
        L.orc_nonempty_rows.restype = C.c_int64
        L.orc_nonempty_rows.argtypes = [vp, C.c_int, vp, vp, vp, vp, C.c_int64]
        L.orc_init_tree_structure.argtypes = [vp, vp, vp]
        L.orc_free_access.argtypes = [vp]
        L.orc_fill_tree.argtypes = [vp, vp, vp, vp, vp]
        L.orc_reconstruct_level.argtypes = [vp, vp, vp, vp, C.c_int, vp]
        L.orc_reconstruct_patch.argtypes = [vp, vp, vp, vp, vp, vp]
        L.orc_convolve_pixels.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp]
        L.orc_validate.restype = C.c_int
        L.orc_validate.argtypes = [vp, vp, vp, C.c_size_t]
        L.orc_restrict_stencil.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp]
        L.orc_convolve.argtypes = [vp, vp, vp, vp, vp, C.c_int, vp]
        L.orc_rl_apr.argtypes = [vp, vp, vp, vp, vp, vp, C.c_int, C.c_double, vp]
        L.orc_generate_spheres.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                           C.c_double, C.c_double, C.c_double, C.c_uint64, C.c_int, vp]
        L.orc_build_apr.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, vp, vp]
        L.orc_free_values.argtypes = [vp]

    def reflect_index(self, i: int, n: int) -> int:
        return self.L.orc_reflect_index(i, n)

    def init_tree_structure(self, leaf, dims) -> Access:
        keep = []
        la = _orc_access(leaf, keep)
        d = np.array(dims, np.int32)
        out = _OrcOwned()
        self.L.orc_init_tree_structure(C.byref(la), d.ctypes.data, C.byref(out))
        n = out.l_max + 1
        res = Access(out.l_min, out.l_max,
                     np.ctypeslib.as_array(out.z_dim, (n,)).copy(), np.ctypeslib.as_array(out.x_dim, (n,)).copy(),
                     np.ctypeslib.as_array(out.y_dim, (n,)).copy(),
                     np.ctypeslib.as_array(out.y_idx, (max(out.n_particles, 1),))[:out.n_particles].copy(),
                     np.ctypeslib.as_array(out.xz_end, (max(out.n_rows, 1),))[:out.n_rows].copy(),
                     np.ctypeslib.as_array(out.level_offset, (n,)).copy())
        self.L.orc_free_access(C.byref(out))
        return res

    def generate_spheres(self, dims, count, rmin, rmax, blur=2.0, seed=42, background=100.0, imin=500.0,
                         imax=2000.0, threads=0) -> np.ndarray:
        """generate_spheres (synthetic.hpp:74-111, no noise), multi-threaded C."""
        threads = threads or os.cpu_count() or 1
        out = np.empty(tuple(int(d) for d in dims), np.float32)
        if self.L.orc_generate_spheres(int(dims[0]), int(dims[1]), int(dims[2]), int(count), C.c_double(rmin),
                                       C.c_double(rmax), C.c_double(background), C.c_double(imin),
                                       C.c_double(imax), C.c_double(blur), C.c_uint64(seed), int(threads),
                                       out.ctypes.data):
            raise MemoryError("orc_generate_spheres failed")
        return out

    def build_apr(self, vol: np.ndarray, rel_error=0.1, threads=0):
        """build_apr (build.hpp:290-312), spheres recipe: (leaf Access, values)."""
        threads = threads or os.cpu_count() or 1
        v = np.ascontiguousarray(vol, np.float32)
        out = _OrcOwned()
        vals = C.POINTER(C.c_float)()
        if self.L.orc_build_apr(v.ctypes.data, v.shape[0], v.shape[1], v.shape[2], C.c_double(rel_error),
                                int(threads), C.byref(out), C.byref(vals)):
            raise MemoryError("orc_build_apr failed")
        n = out.l_max + 1
        res = Access(out.l_min, out.l_max,
                     np.ctypeslib.as_array(out.z_dim, (n,)).copy(), np.ctypeslib.as_array(out.x_dim, (n,)).copy(),
                     np.ctypeslib.as_array(out.y_dim, (n,)).copy(),
                     np.ctypeslib.as_array(out.y_idx, (max(out.n_particles, 1),))[:out.n_particles].copy(),
                     np.ctypeslib.as_array(out.xz_end, (max(out.n_rows, 1),))[:out.n_rows].copy(),
                     np.ctypeslib.as_array(out.level_offset, (n,)).copy())
        values = np.ctypeslib.as_array(vals, (max(out.n_particles, 1),))[:out.n_particles].copy()
        self.L.orc_free_access(C.byref(out))
        self.L.orc_free_values(vals)
        return res, values

    def build_spheres(self, n, count, rmin, rmax, blur=2.0, seed=42, rel_error=0.1, threads=0):
        """generate_spheres + build_apr of an n^3 (or (nz, nx, ny)) sphere scene."""
        dims = (n, n, n) if np.isscalar(n) else tuple(n)
        vol = self.generate_spheres(dims, count, rmin, rmax, blur, seed, threads=threads)
        acc, values = self.build_apr(vol, rel_error, threads)
        del vol
        return acc, values

    def fill_tree(self, leaf, tree, dims, values) -> np.ndarray:
        keep = []
        la, ta = _orc_access(leaf, keep), _orc_access(tree, keep)
        d = np.array(dims, np.int32)
        v = np.ascontiguousarray(values, np.float32)
        out = np.zeros(ta.n_particles, np.float32)
        st = self.L.orc_fill_tree(C.byref(la), C.byref(ta), d.ctypes.data, _p(v), _p(out))
        if st:
            raise RuntimeError(f"orc_fill_tree status {st}")
        return out

    def nonempty_rows(self, leaf, level: int):
        keep = []
        la = _orc_access(leaf, keep)
        n = self.L.orc_nonempty_rows(C.byref(la), level, None, None, None, None, C.c_int64(0))
        z, x = np.zeros(n, np.int32), np.zeros(n, np.int32)
        y0, y1 = np.zeros(n, np.uint16), np.zeros(n, np.uint16)
        self.L.orc_nonempty_rows(C.byref(la), level, _p(z), _p(x), _p(y0), _p(y1), C.c_int64(n))
        return z, x, y0, y1

    def reconstruct_level(self, leaf, tree, values, tree_values, l: int) -> np.ndarray:
        keep = []
        la, ta = _orc_access(leaf, keep), _orc_access(tree, keep)
        a = as_access(leaf)
        out = np.zeros((int(a.z_dim[l]), int(a.x_dim[l]), int(a.y_dim[l])), np.float32)
        v = np.ascontiguousarray(values, np.float32)
        tv = None if tree_values is None else np.ascontiguousarray(tree_values, np.float32)
        self.L.orc_reconstruct_level(C.byref(la), _p(v), C.byref(ta), None if tv is None else _p(tv), l,
                                     out.ctypes.data)
        return out

    def convolve_pixels(self, vol: np.ndarray, w: np.ndarray, k3, pad: int) -> np.ndarray:
        v = np.ascontiguousarray(vol, np.float32)
        ww = np.ascontiguousarray(w, np.float32).reshape(-1)
        out = np.empty_like(v)
        nz, nx, ny = v.shape
        self.L.orc_convolve_pixels(v.ctypes.data, nz, nx, ny, ww.ctypes.data, int(k3[0]), int(k3[1]), int(k3[2]),
                                   int(pad), out.ctypes.data)
        return out

    def validate(self, leaf, dims):
        """validate (apr.hpp:61-134): (ok, message)."""
        keep = []
        la = _orc_access(leaf, keep)
        dm = np.array([int(v) for v in dims], np.int32)
        buf = C.create_string_buffer(512)
        ok = self.L.orc_validate(C.byref(la), dm.ctypes.data, buf, 512)
        return bool(ok), buf.value.decode()

    def reconstruct_patch(self, leaf, tree, values, tree_values, spec) -> np.ndarray:
        """spec: (level, z_begin, z_end, x_begin, x_end, pad, pad_mode)."""
        keep = []
        la, ta = _orc_access(leaf, keep), _orc_access(tree, keep)
        a = as_access(leaf)
        l, zb, ze, xb, xe, pad, _ = (int(v) for v in spec)
        out = np.zeros((ze - zb + 2 * pad, xe - xb + 2 * pad, int(a.y_dim[l]) + 2 * pad), np.float32)
        v = np.ascontiguousarray(values, np.float32)
        tv = None if tree_values is None else np.ascontiguousarray(tree_values, np.float32)
        sp = np.array(spec, np.int32)
        self.L.orc_reconstruct_patch(C.byref(la), _p(v), C.byref(ta), None if tv is None else _p(tv), _p(sp),
                                     out.ctypes.data)
        return out

    def restrict_stencil(self, w: np.ndarray, k3, delta: int):
        w = np.ascontiguousarray(w, np.float32).reshape(-1)
        ok = (C.c_int * 3)()
        self.L.orc_restrict_stencil(w.ctypes.data, k3[0], k3[1], k3[2], delta, ok, None)
        out = np.zeros(ok[0] * ok[1] * ok[2], np.float32)
        self.L.orc_restrict_stencil(w.ctypes.data, k3[0], k3[1], k3[2], delta, ok, out.ctypes.data)
        return (ok[0], ok[1], ok[2]), out

    @staticmethod
    def _pyr(levels, l_min: int, keep: list) -> _OrcPyr:
        """levels: list of (k3, weights) for l_min..l_max"""
        k3 = np.array([list(k) for k, _ in levels], np.int32).reshape(-1)
        w = np.concatenate([np.asarray(ws, np.float32).reshape(-1) for _, ws in levels])
        off = np.cumsum([0] + [int(np.prod(k)) for k, _ in levels[:-1]]).astype(np.uint64)
        keep += [k3, w, off]
        p = _OrcPyr()
        p.l_min, p.l_max = l_min, l_min + len(levels) - 1
        p.k3, p.w, p.off = k3.ctypes.data, w.ctypes.data, off.ctypes.data
        return p

    def convolve(self, leaf, tree, values, tree_values, levels, l_min: int, pad: int) -> np.ndarray:
        keep = []
        la, ta = _orc_access(leaf, keep), _orc_access(tree, keep)
        p = self._pyr(levels, l_min, keep)
        v = np.ascontiguousarray(values, np.float32)
        tv = np.ascontiguousarray(tree_values, np.float32)
        out = np.zeros(la.n_particles, np.float32)
        st = self.L.orc_convolve(C.byref(la), C.byref(ta), _p(v), _p(tv), C.byref(p), pad, _p(out))
        if st:
            raise RuntimeError(f"orc_convolve status {st}")
        return out

    def restricted_levels(self, w, k3, l_min: int, l_max: int):
        return [self.restrict_stencil(w, k3, l_max - l) for l in range(l_min, l_max + 1)]

    def rl_apr(self, leaf, tree, dims, observed, w, k3, iterations: int, eps: float = 0.0) -> np.ndarray:
        """rl_apr with normalized_psf / flip / restricted pyramids / rl_epsilon
        prepared here exactly as deconv.hpp:75-93 does."""
        a = as_access(leaf)
        w = np.asarray(w, np.float32).reshape(-1)
        s = 0.0
        for x in w.tolist():
            s += x
        wn = np.array([np.float32(x / s) for x in w.tolist()], np.float32)
        wt = wn.reshape(k3)[::-1, ::-1, ::-1].reshape(-1).copy()
        u = np.maximum(np.asarray(observed, np.float32), np.float32(0))
        mean = 0.0
        for x in u.tolist():
            mean += x
        mean /= max(u.size, 1)
        if eps <= 0:
            eps = 1e-6 * max(mean, 1e-30)
        keep = []
        la, ta = _orc_access(leaf, keep), _orc_access(tree, keep)
        pw = self._pyr(self.restricted_levels(wn, k3, a.l_min, a.l_max), a.l_min, keep)
        pwt = self._pyr(self.restricted_levels(wt, k3, a.l_min, a.l_max), a.l_min, keep)
        d = np.array(dims, np.int32)
        obs = np.ascontiguousarray(observed, np.float32)
        out = np.zeros(la.n_particles, np.float32)
        st = self.L.orc_rl_apr(C.byref(la), C.byref(ta), d.ctypes.data, _p(obs), C.byref(pw), C.byref(pwt),
                               iterations, C.c_double(eps), _p(out))
        if st:
            raise RuntimeError(f"orc_rl_apr status {st}")
        return out


# ---------------------------------------------------------- real reference ----
def ref_available() -> bool:
    return os.path.exists(REF_SO)


class RefApr:
    def __init__(self, lib: "Ref", h: int):
        self.lib, self.h = lib, h

    def __del__(self):
        try:
            self.lib.L.ref_apr_free(self.h)
        except Exception:
            pass

    def access(self, which: int) -> Access:
        L = self.lib.L
        info = (C.c_int64 * 4)()
        L.ref_apr_info(self.h, which, info)
        l_min, l_max, n_p, n_r = (int(v) for v in info)
        n = l_max + 1
        y = np.zeros(n_p, np.uint16)
        e = np.zeros(n_r, np.uint64)
        lo = np.zeros(n, np.uint64)
        zd, xd, yd = (np.zeros(n, np.int32) for _ in range(3))
        L.ref_apr_copy(self.h, which, _p(y), _p(e), lo.ctypes.data, zd.ctypes.data, xd.ctypes.data, yd.ctypes.data)
        return Access(l_min, l_max, zd, xd, yd, y, e, lo)

    @property
    def leaf(self) -> Access:
        return self.access(0)

    @property
    def tree(self) -> Access:
        return self.access(1)

    @property
    def dims(self):
        d = (C.c_int * 3)()
        self.lib.L.ref_apr_dims(self.h, d)
        return (d[0], d[1], d[2])

    def values(self) -> np.ndarray:
        n = self.lib.L.ref_apr_values(self.h, None)
        out = np.zeros(n, np.float32)
        self.lib.L.ref_apr_values(self.h, _p(out))
        return out

    def n_particles(self) -> int:
        return self.leaf.y_idx.size


class Ref:
    """The unmodified reference (aprkit) compiled into oracle/_ref/libaprref.so."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise RuntimeError(f"reference library not built: {path}")
        L = C.CDLL(path)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_rng_new.restype = vp
        L.ref_rng_new.argtypes = [C.c_uint64]
        L.ref_rng_free.argtypes = [vp]
        L.ref_rng_next_u64.restype = C.c_uint64
        L.ref_rng_next_u64.argtypes = [vp]
        L.ref_rng_uniform.restype = C.c_double
        L.ref_rng_uniform.argtypes = [vp, C.c_double, C.c_double]
        L.ref_rng_uniform_int.restype = C.c_int64
        L.ref_rng_uniform_int.argtypes = [vp, C.c_int64, C.c_int64]
        L.ref_random_apr.restype = vp
        L.ref_random_apr.argtypes = [vp, C.c_int, C.c_int]
        L.ref_random_values.argtypes = [vp, C.c_uint64, C.c_double, C.c_double, vp]
        L.ref_random_stencil.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, vp]
        L.ref_apr_from_targets.restype = vp
        L.ref_apr_from_targets.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_apr_from_arrays.restype = vp
        L.ref_apr_from_arrays.argtypes = [C.c_int, C.c_int, vp, vp, vp, vp, C.c_uint64, vp, C.c_uint64, vp,
                                          C.c_int, C.c_int, C.c_int]
        L.ref_build_spheres.restype = vp
        L.ref_build_spheres.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                        C.c_double, C.c_uint64, C.c_double, C.c_int]
        L.ref_generate_spheres.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                           C.c_double, C.c_uint64, vp]
        L.ref_build_apr.restype = vp
        L.ref_build_apr.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int]
        L.ref_build_apr_params.restype = vp
        L.ref_build_apr_params.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_double, C.c_int,
                                           C.c_double, C.c_int, C.c_int, C.c_int]
        L.ref_sample_particles.argtypes = [vp, vp, vp]
        L.ref_apr_free.argtypes = [vp]
        L.ref_apr_info.argtypes = [vp, C.c_int, vp]
        L.ref_apr_dims.argtypes = [vp, vp]
        L.ref_apr_copy.argtypes = [vp, C.c_int, vp, vp, vp, vp, vp, vp]
        L.ref_apr_values.restype = C.c_uint64
        L.ref_apr_values.argtypes = [vp, vp]
        L.ref_validate.argtypes = [vp]
        L.ref_fill_tree.argtypes = [vp, vp, C.c_int, vp]
        L.ref_nonempty_row_index.restype = C.c_int64
        L.ref_nonempty_row_index.argtypes = [vp, C.c_int, vp, vp, vp, vp]
        L.ref_make_pyramid.restype = vp
        L.ref_make_pyramid.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_explicit_pyramid.restype = vp
        L.ref_explicit_pyramid.argtypes = [vp, vp, C.c_int, C.c_int]
        L.ref_pyramid_free.argtypes = [vp]
        L.ref_pyramid_level.argtypes = [vp, C.c_int, vp, vp]
        L.ref_restrict_stencil.argtypes = [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp]
        L.ref_gaussian_stencil.argtypes = [C.c_double, C.c_int, vp, vp]
        L.ref_box_stencil.argtypes = [C.c_int, vp]
        L.ref_convolve.argtypes = [vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp]
        L.ref_reconstruct_level.argtypes = [vp, vp, vp, C.c_int, vp]
        L.ref_reconstruct_full.argtypes = [vp, vp, vp]
        L.ref_save_apr.argtypes = [vp, vp, C.c_char_p]
        L.ref_convolve_pixels.argtypes = [vp, C.c_int, C.c_int, C.c_int, vp, C.c_int, C.c_int, C.c_int, C.c_int, vp]
        L.ref_load_apr.restype = C.c_int
        L.ref_load_apr.argtypes = [C.c_char_p, C.POINTER(vp), vp, C.c_uint64]
        L.ref_validate_arrays.restype = C.c_int
        L.ref_validate_arrays.argtypes = [C.c_int, C.c_int, vp, vp, vp, vp, C.c_uint64, vp, C.c_uint64, vp,
                                          C.c_int, C.c_int, C.c_int, vp, C.c_uint64]
        L.ref_reconstruct_patch.argtypes = [vp, vp, vp, vp, vp]
        L.ref_rl_apr.argtypes = [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, vp]
        L.ref_resolve_threads.argtypes = [C.c_int]
        self.L = L

    def err(self) -> str:
        return self.L.ref_last_error().decode()

    def _chk(self, st: int):
        if st:
            raise RuntimeError(f"reference status {st}: {self.err()}")

    # rng + helpers
    def rng(self, seed: int):
        return C.c_void_p(self.L.ref_rng_new(seed))

    def random_apr(self, rng, min_dim: int = 4, max_dim: int = 40) -> RefApr:
        return RefApr(self, self.L.ref_random_apr(rng, min_dim, max_dim))

    def random_values(self, rng, n: int, lo: float = 0.0, hi: float = 1000.0) -> np.ndarray:
        out = np.zeros(n, np.float32)
        self.L.ref_random_values(rng, n, lo, hi, _p(out))
        return out

    def random_stencil(self, rng, kz: int, kx: int, ky: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
        out = np.zeros(kz * kx * ky, np.float32)
        self.L.ref_random_stencil(rng, kz, kx, ky, lo, hi, out.ctypes.data)
        return out

    def apr_from_targets(self, targets: np.ndarray, l_min: int, l_max: int) -> RefApr:
        t = np.ascontiguousarray(targets, np.int32)
        nz, nx, ny = t.shape
        h = self.L.ref_apr_from_targets(t.ctypes.data, nz, nx, ny, l_min, l_max)
        if not h:
            raise RuntimeError(self.err())
        return RefApr(self, h)

    def apr_from_arrays(self, leaf, dims) -> RefApr:
        a = as_access(leaf)
        h = self.L.ref_apr_from_arrays(a.l_min, a.l_max, a.z_dim.ctypes.data, a.x_dim.ctypes.data,
                                       a.y_dim.ctypes.data, _p(a.y_idx), a.y_idx.size, _p(a.xz_end), a.xz_end.size,
                                       a.level_offset.ctypes.data, dims[0], dims[1], dims[2])
        if not h:
            raise RuntimeError(self.err())
        return RefApr(self, h)

    def build_spheres(self, n, count, rmin, rmax, blur=2.0, noise=0.0, seed=42, rel_error=0.1, threads=0) -> RefApr:
        nz, nx, ny = (n, n, n) if np.isscalar(n) else n
        h = self.L.ref_build_spheres(nz, nx, ny, count, rmin, rmax, blur, noise, seed, rel_error, threads)
        if not h:
            raise RuntimeError(self.err())
        return RefApr(self, h)

    def generate_spheres(self, dims, count, rmin, rmax, blur=2.0, noise=0.0, seed=42) -> np.ndarray:
        out = np.zeros(dims, np.float32)
        self._chk(self.L.ref_generate_spheres(dims[0], dims[1], dims[2], count, rmin, rmax, blur, noise, seed,
                                              out.ctypes.data))
        return out

    def build_apr(self, vol: np.ndarray, rel_error=0.1, threads=0) -> RefApr:
        v = np.ascontiguousarray(vol, np.float32)
        h = self.L.ref_build_apr(v.ctypes.data, v.shape[0], v.shape[1], v.shape[2], rel_error, threads)
        if not h:
            raise RuntimeError(self.err())
        return RefApr(self, h)

    def build_apr_params(self, vol: np.ndarray, rel_error=0.1, sigma_mode=0, sigma_value=1.0, sigma_window=2,
                         sigma_floor=0.0, gradient_mode=0, smoothing_passes=0, threads=0) -> RefApr:
        """build_apr (build.hpp:290-312) with every BuildParams field."""
        v = np.ascontiguousarray(vol, np.float32)
        h = self.L.ref_build_apr_params(v.ctypes.data, v.shape[0], v.shape[1], v.shape[2], rel_error, sigma_mode,
                                        sigma_value, sigma_window, sigma_floor, gradient_mode, smoothing_passes,
                                        threads)
        if not h:
            raise RuntimeError(self.err())
        return RefApr(self, h)

    def validate(self, apr: RefApr) -> bool:
        return bool(self.L.ref_validate(apr.h))

    def fill_tree(self, apr: RefApr, values, threads: int = 0) -> np.ndarray:
        v = np.ascontiguousarray(values, np.float32)
        out = np.zeros(apr.tree.y_idx.size, np.float32)
        self._chk(self.L.ref_fill_tree(apr.h, _p(v), threads, _p(out)))
        return out

    def nonempty_rows(self, apr: RefApr, level: int):
        n = self.L.ref_nonempty_row_index(apr.h, level, None, None, None, None)
        z, x = np.zeros(n, np.int32), np.zeros(n, np.int32)
        y0, y1 = np.zeros(n, np.uint16), np.zeros(n, np.uint16)
        if n:
            self.L.ref_nonempty_row_index(apr.h, level, z.ctypes.data, x.ctypes.data, y0.ctypes.data, y1.ctypes.data)
        return z, x, y0, y1

    def make_pyramid(self, w, k3, l_min, l_max, mode=0):
        w = np.ascontiguousarray(w, np.float32).reshape(-1)
        h = self.L.ref_make_pyramid(w.ctypes.data, k3[0], k3[1], k3[2], l_min, l_max, mode)
        if not h:
            raise RuntimeError(self.err())
        return RefPyramid(self, h, l_min, l_max)

    def explicit_pyramid(self, levels, l_min):
        k3 = np.array([list(k) for k, _ in levels], np.int32).reshape(-1)
        w = np.concatenate([np.asarray(x, np.float32).reshape(-1) for _, x in levels])
        h = self.L.ref_explicit_pyramid(w.ctypes.data, k3.ctypes.data, l_min, l_min + len(levels) - 1)
        if not h:
            raise RuntimeError(self.err())
        return RefPyramid(self, h, l_min, l_min + len(levels) - 1)

    def restrict_stencil(self, w, k3, delta):
        w = np.ascontiguousarray(w, np.float32).reshape(-1)
        ok = (C.c_int * 3)()
        self._chk(self.L.ref_restrict_stencil(w.ctypes.data, k3[0], k3[1], k3[2], delta, ok, None))
        out = np.zeros(ok[0] * ok[1] * ok[2], np.float32)
        self._chk(self.L.ref_restrict_stencil(w.ctypes.data, k3[0], k3[1], k3[2], delta, ok, out.ctypes.data))
        return (ok[0], ok[1], ok[2]), out

    def gaussian_stencil(self, sigma, size=0):
        k = C.c_int()
        self._chk(self.L.ref_gaussian_stencil(sigma, size, C.byref(k), None))
        out = np.zeros(k.value ** 3, np.float32)
        self._chk(self.L.ref_gaussian_stencil(sigma, size, C.byref(k), out.ctypes.data))
        return (k.value,) * 3, out

    def convolve(self, apr: RefApr, values, tree_values, pyr: "RefPyramid", pad=1, threads=0, row_skip=True):
        v = np.ascontiguousarray(values, np.float32)
        tv = np.ascontiguousarray(tree_values, np.float32)
        out = np.zeros(v.size, np.float32)
        self._chk(self.L.ref_convolve(apr.h, _p(v), _p(tv), pyr.h, pad, threads, 1 if row_skip else 0, _p(out)))
        return out

    def reconstruct_level(self, apr: RefApr, values, tree_values, l):
        a = apr.leaf
        out = np.zeros((int(a.z_dim[l]), int(a.x_dim[l]), int(a.y_dim[l])), np.float32)
        v = np.ascontiguousarray(values, np.float32)
        tv = None if tree_values is None else np.ascontiguousarray(tree_values, np.float32)
        self._chk(self.L.ref_reconstruct_level(apr.h, _p(v), None if tv is None else _p(tv), l, out.ctypes.data))
        return out

    def convolve_pixels(self, vol: np.ndarray, w: np.ndarray, k3, pad: int) -> np.ndarray:
        v = np.ascontiguousarray(vol, np.float32)
        ww = np.ascontiguousarray(w, np.float32).reshape(-1)
        out = np.empty_like(v)
        nz, nx, ny = v.shape
        self._chk(self.L.ref_convolve_pixels(v.ctypes.data, nz, nx, ny, ww.ctypes.data, int(k3[0]), int(k3[1]),
                                             int(k3[2]), int(pad), out.ctypes.data))
        return out

    def save_apr(self, apr: "RefApr", values, path: str):
        v = np.ascontiguousarray(values, np.float32)
        self._chk(self.L.ref_save_apr(apr.h, _p(v), path.encode()))

    def load_apr(self, path: str):
        """(kind, message, RefApr or None): kind 0 ok, 1 IoError, 2 BadFormatError, 3 TruncatedFileError."""
        h = C.c_void_p()
        buf = C.create_string_buffer(512)
        kind = self.L.ref_load_apr(path.encode(), C.byref(h), buf, 512)
        return kind, buf.value.decode(), (RefApr(self, h.value) if kind == 0 else None)

    def validate_arrays(self, leaf, dims):
        """validate (apr.hpp:61-134) of a leaf access: (ok, message)."""
        a = as_access(leaf)
        buf = C.create_string_buffer(512)
        ok = self.L.ref_validate_arrays(a.l_min, a.l_max, a.z_dim.ctypes.data, a.x_dim.ctypes.data,
                                        a.y_dim.ctypes.data, _p(a.y_idx), a.y_idx.size, _p(a.xz_end),
                                        a.xz_end.size, a.level_offset.ctypes.data, int(dims[0]), int(dims[1]),
                                        int(dims[2]), buf, 512)
        return bool(ok), buf.value.decode()

    def reconstruct_full(self, apr: RefApr, values):
        a = apr.leaf
        l = a.l_max
        out = np.zeros((int(a.z_dim[l]), int(a.x_dim[l]), int(a.y_dim[l])), np.float32)
        v = np.ascontiguousarray(values, np.float32)
        self._chk(self.L.ref_reconstruct_full(apr.h, _p(v), out.ctypes.data))
        return out

    def reconstruct_patch(self, apr: RefApr, values, tree_values, spec):
        a = apr.leaf
        l, zb, ze, xb, xe, pad, _ = (int(v) for v in spec)
        out = np.zeros((ze - zb + 2 * pad, xe - xb + 2 * pad, int(a.y_dim[l]) + 2 * pad), np.float32)
        v = np.ascontiguousarray(values, np.float32)
        tv = None if tree_values is None else np.ascontiguousarray(tree_values, np.float32)
        sp = np.array(spec, np.int32)
        self._chk(self.L.ref_reconstruct_patch(apr.h, _p(v), None if tv is None else _p(tv), _p(sp),
                                               out.ctypes.data))
        return out

    def rl_apr(self, apr: RefApr, observed, w, k3, iterations, epsilon=0.0, threads=0):
        obs = np.ascontiguousarray(observed, np.float32)
        w = np.ascontiguousarray(w, np.float32).reshape(-1)
        out = np.zeros(obs.size, np.float32)
        self._chk(self.L.ref_rl_apr(apr.h, _p(obs), w.ctypes.data, k3[0], k3[1], k3[2], iterations, epsilon,
                                    threads, _p(out)))
        return out

    def resolve_threads(self, requested=0) -> int:
        return self.L.ref_resolve_threads(requested)


class RefPyramid:
    def __init__(self, lib: Ref, h: int, l_min: int, l_max: int):
        self.lib, self.h, self.l_min, self.l_max = lib, h, l_min, l_max

    def __del__(self):
        try:
            self.lib.L.ref_pyramid_free(self.h)
        except Exception:
            pass

    def level(self, l: int):
        k3 = (C.c_int * 3)()
        self.lib._chk(self.lib.L.ref_pyramid_level(self.h, l, k3, None))
        w = np.zeros(k3[0] * k3[1] * k3[2], np.float32)
        self.lib._chk(self.lib.L.ref_pyramid_level(self.h, l, k3, w.ctypes.data))
        return (k3[0], k3[1], k3[2]), w

    def levels(self):
        return [self.level(l) for l in range(self.l_min, self.l_max + 1)]
