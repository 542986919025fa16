"""TEST INFRASTRUCTURE: Python loaders for the two CPU oracles.

  * ``OracleC``   -- oracle/_build/liboracle.so, the plain-C restatement
                     (oracle/edgealign_oracle.c).
  * ``ReferenceLib`` -- oracle/_ref/libedgealign_ref.so, the reference itself
                     compiled from /root/reference/proj/src (oracle/Makefile)
                     behind the C shim oracle/ref_shim.cpp.

Both expose the same Python surface so tests can arbitrate the CUDA path
against either.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / reference legs may import this module.
"""
import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from paper_2112_05576_b200 import abi
from paper_2112_05576_b200.errors import raise_for_status

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libedgealign_ref.so")
REF_SRC = "/root/reference/proj"

_dp = C.POINTER(C.c_double)


def _ptr(a):
    return a.ctypes.data_as(_dp)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class EdgeModel:
    """edgealign::EdgeModel (edge_model.h:40-45); points is (n, 5) float64."""
    points: np.ndarray
    centroid_x: float
    centroid_y: float
    source_level: int = 0

    def as_c(self):
        pts = np.ascontiguousarray(self.points, dtype=np.float64)
        return pts, pts.ctypes.data_as(C.POINTER(abi.EdgePoint)), len(pts)


def build_oracle(force=False):
    if force or not os.path.exists(ORACLE_SO):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return ORACLE_SO


def build_reference(force=False):
    """Compile the reference from its own sources (needs /root/reference)."""
    if force or not os.path.exists(REF_SO):
        if not os.path.isdir(REF_SRC):
            return None
        subprocess.run(["make", "-s", "-C", HERE, "ref", f"-j{os.cpu_count() or 4}"],
                       check=True)
    return REF_SO


class _Base:
    prefix = ""

    def __init__(self, path):
        self.lib = C.CDLL(path)
        p = self.prefix
        getattr(self.lib, p + "last_error").restype = C.c_char_p
        getattr(self.lib, p + "last_error_value").restype = C.c_double

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _check(self, st):
        if st != abi.EA_OK:
            raise_for_status(st, self._fn("last_error")(), self._fn("last_error_value")())

    # ---- geometry ----------------------------------------------------------
    def grid_counts(self, g):
        out = abi.GridCounts()
        self._check(self._fn("grid_counts")(C.byref(g), C.byref(out)))
        return (out.nx, out.ny, out.nt)

    def pose_at(self, g, index):
        out = abi.Pose()
        self._check(self._fn("pose_at")(C.byref(g), C.c_uint64(index), C.byref(out)))
        return out.astuple()

    # ---- image ---------------------------------------------------------------
    def downsample(self, img):
        img = _f64(img)
        h, w = img.shape
        out = np.zeros((max(h // 2, 1), max(w // 2, 1)))
        self._check(self._fn("downsample")(_ptr(img), w, h, _ptr(out)))
        return out

    def max_pyramid_levels(self, w, h):
        return self._fn("max_pyramid_levels")(w, h)

    def build_pyramid(self, img, levels):
        img = _f64(img)
        h, w = img.shape
        dims = [(w >> l, h >> l) for l in range(max(levels, 1))]
        total = sum(a * b for a, b in dims)
        out = np.zeros(total)
        self._check(self._fn("build_pyramid")(_ptr(img), w, h, levels, _ptr(out)))
        res, off = [], 0
        for (lw, lh) in dims:
            res.append(out[off: off + lw * lh].reshape(lh, lw).copy())
            off += lw * lh
        return res

    def compute_gradients(self, img):
        img = _f64(img)
        h, w = img.shape
        gx, gy, mag = (np.zeros((h, w)) for _ in range(3))
        self._check(self._fn("compute_gradients")(_ptr(img), w, h, _ptr(gx), _ptr(gy),
                                                  _ptr(mag)))
        return gx, gy, mag

    # ---- template side ---------------------------------------------------------
    def extract_edge_model(self, field, th, level=0):
        gx, gy, mag = (_f64(a) for a in field)
        h, w = mag.shape
        cap = w * h
        pts = np.zeros((max(cap, 1), 5))
        n, cx, cy = C.c_int(), C.c_double(), C.c_double()
        t = abi.EdgeThresholds(*th)
        self._check(self._fn("extract_edge_model")(
            _ptr(gx), _ptr(gy), _ptr(mag), w, h, C.byref(t), level,
            pts.ctypes.data_as(C.POINTER(abi.EdgePoint)), cap, C.byref(n), C.byref(cx),
            C.byref(cy)))
        return EdgeModel(pts[: n.value].copy(), cx.value, cy.value, level)

    # ---- similarity ------------------------------------------------------------
    def rotate_model(self, points, theta):
        pts = np.ascontiguousarray(points, dtype=np.float64)
        n = len(pts)
        px, py, dx, dy = (np.zeros(n) for _ in range(4))
        self._check(self._fn("rotate_model")(pts.ctypes.data_as(C.POINTER(abi.EdgePoint)), n,
                                             C.c_double(theta), _ptr(px), _ptr(py), _ptr(dx),
                                             _ptr(dy)))
        return px, py, dx, dy

    def pose_score(self, points, pose, field, params):
        pts = np.ascontiguousarray(points, dtype=np.float64)
        gx, gy, mag = (_f64(a) for a in field)
        h, w = mag.shape
        v, nin = C.c_double(), C.c_int()
        self._check(self._fn("pose_score")(pts.ctypes.data_as(C.POINTER(abi.EdgePoint)),
                                           len(pts), C.byref(abi.Pose(*pose)), _ptr(gx),
                                           _ptr(gy), _ptr(mag), w, h, C.byref(params),
                                           C.byref(v), C.byref(nin)))
        return v.value, nin.value

    def render_template(self, template_id, size):
        tid = abi.TEMPLATE_IDS[template_id] if isinstance(template_id, str) else template_id
        out = np.zeros((max(size, 1), max(size, 1)))
        self._check(self._fn("render_template")(tid, size, _ptr(out)))
        return out

    def compose_scene(self, spec):
        canvas = np.zeros((spec.canvas_height, spec.canvas_width))
        tmpl = np.zeros((spec.template_size, spec.template_size))
        pose, occ = abi.Pose(), C.c_double()
        self._check(self._fn("compose_scene")(C.byref(spec), _ptr(canvas), _ptr(tmpl),
                                              C.byref(pose), C.byref(occ)))
        return canvas, tmpl, pose.astuple(), occ.value

    def prepare_model(self, tmpl_img, level=0, thresholds=None):
        f = self.compute_gradients(tmpl_img)
        th = thresholds if thresholds is not None else self.default_thresholds(f)
        return self.extract_edge_model(f, th, level)


class OracleC(_Base):
    """The plain-C restatement (oracle/edgealign_oracle.c)."""
    prefix = "orc_"

    def __init__(self, path=None):
        super().__init__(path or build_oracle())

    def default_thresholds(self, field):
        mag = _f64(field[2])
        h, w = mag.shape
        t = abi.EdgeThresholds()
        self._check(self.lib.orc_default_thresholds(_ptr(mag), w, h, C.byref(t)))
        return (t.low, t.high)

    def point_vote(self, dir_x, dir_y, field, cx, cy, params):
        gx, gy, mag = (_f64(a) for a in field)
        h, w = mag.shape
        out = C.c_double()
        self._check(self.lib.orc_point_vote(C.c_double(dir_x), C.c_double(dir_y), _ptr(gx),
                                            _ptr(gy), _ptr(mag), w, h, cx, cy, C.byref(params),
                                            C.byref(out)))
        return out.value

    def search_topk(self, points, field, grid, params, k, threads=0, it_range=(0, 0)):
        pts = np.ascontiguousarray(points, dtype=np.float64)
        gx, gy, mag = (_f64(a) for a in field)
        h, w = mag.shape
        out = (abi.ScoredPose * max(k, 1))()
        n = C.c_int()
        self._check(self.lib.orc_search_topk(
            pts.ctypes.data_as(C.POINTER(abi.EdgePoint)), len(pts), _ptr(gx), _ptr(gy),
            _ptr(mag), w, h, C.byref(grid), C.byref(params), k, C.c_uint64(it_range[0]),
            C.c_uint64(it_range[1]), threads, out, C.byref(n)))
        return list(out[: n.value])

    def exhaustive_search(self, points, field, grid, params, threads=0):
        return self.search_topk(points, field, grid, params, 1, threads)[0]

    def score_map(self, points, field, grid, params, max_cells):
        pts = np.ascontiguousarray(points, dtype=np.float64)
        gx, gy, mag = (_f64(a) for a in field)
        h, w = mag.shape
        total = 1
        try:
            total = int(np.prod(self.grid_counts(grid)))
        except Exception:
            pass
        out = np.zeros(max(min(total, max_cells), 1))
        self._check(self.lib.orc_score_map(pts.ctypes.data_as(C.POINTER(abi.EdgePoint)),
                                           len(pts), _ptr(gx), _ptr(gy), _ptr(mag), w, h,
                                           C.byref(grid), C.byref(params),
                                           C.c_uint64(max_cells), _ptr(out)))
        return out[:total]

    def prepare_levels(self, tmpl_pyr, work_pyr, cfg):
        """search.cpp:208-238 (Python orchestration of the C primitives)."""
        from paper_2112_05576_b200.errors import EmptyModelError, InvalidArgument
        L = cfg.num_levels
        if L < 1:
            raise InvalidArgument("num_levels must be >= 1")
        if len(tmpl_pyr) < L or len(work_pyr) < L:
            raise InvalidArgument(f"pyramids must provide {L} levels")
        models, fields = [], []
        for level in range(L):
            tf = self.compute_gradients(tmpl_pyr[level])
            th = ((cfg.thresholds.low, cfg.thresholds.high) if cfg.has_thresholds
                  else self.default_thresholds(tf))
            try:
                models.append(self.extract_edge_model(tf, th, level))
            except EmptyModelError as e:
                raise EmptyModelError(
                    f"edge model extraction failed at pyramid level {level}: {e}",
                    e.max_magnitude)
            fields.append(self.compute_gradients(work_pyr[level]))
        return models, fields

    def search_levels(self, models, fields, cfg, threads=0):
        L = len(models)
        keep = []
        mp = (C.POINTER(abi.EdgePoint) * L)()
        mn = (C.c_int * L)()
        gxs, gys, mags = (_dp * L)(), (_dp * L)(), (_dp * L)()
        dims = (C.c_int * (2 * L))()
        for l, (m, f) in enumerate(zip(models, fields)):
            pts = np.ascontiguousarray(m.points, dtype=np.float64)
            gx, gy, mag = (_f64(a) for a in f)
            keep += [pts, gx, gy, mag]
            mp[l] = pts.ctypes.data_as(C.POINTER(abi.EdgePoint))
            mn[l] = len(pts)
            gxs[l], gys[l], mags[l] = _ptr(gx), _ptr(gy), _ptr(mag)
            dims[2 * l], dims[2 * l + 1] = mag.shape[1], mag.shape[0]
        out = abi.Outcome()
        self._check(self.lib.orc_search_levels(L, mp, mn, gxs, gys, mags, dims, C.byref(cfg),
                                               threads, C.byref(out)))
        return out

    def coarse_to_fine(self, tmpl_pyr, work_pyr, cfg, threads=0):
        models, fields = self.prepare_levels(tmpl_pyr, work_pyr, cfg)
        return self.search_levels(models, fields, cfg, threads)


class ReferenceLib(_Base):
    """The reference library itself (oracle/_ref), behind oracle/ref_shim.cpp."""
    prefix = "eref_"

    def __init__(self, path=None):
        path = path or build_reference()
        if path is None or not os.path.exists(path):
            raise FileNotFoundError("oracle/_ref/libedgealign_ref.so is not built")
        super().__init__(path)

    def set_isa(self, isa):
        self._check(self.lib.eref_set_isa(isa))

    # ---- Netpbm codecs (image.cpp:26-219) ---------------------------------
    def luminance_to_byte(self, v):
        self.lib.eref_luminance_to_byte.argtypes = [C.c_double]
        return int(self.lib.eref_luminance_to_byte(float(v)))

    def load_pgm(self, data):
        data = bytes(data)
        w, h = C.c_int(), C.c_int()
        self.lib.eref_load_pgm.argtypes = [C.c_char_p, C.c_size_t, C.c_void_p, C.c_size_t,
                                           C.POINTER(C.c_int), C.POINTER(C.c_int)]
        self._check(self.lib.eref_load_pgm(data, len(data), None, 0, C.byref(w), C.byref(h)))
        out = np.zeros((h.value, w.value))
        self._check(self.lib.eref_load_pgm(data, len(data), out.ctypes.data, out.size,
                                           C.byref(w), C.byref(h)))
        return out

    def _save(self, name, img, extra):
        img = _f64(img)
        h, w = img.shape
        n = C.c_size_t()
        fn = getattr(self.lib, name)
        self._check(fn(_ptr(img), w, h, *extra, None, 0, C.byref(n)))
        out = (C.c_ubyte * n.value)()
        self._check(fn(_ptr(img), w, h, *extra, out, n.value, C.byref(n)))
        return bytes(out)

    def save_pgm(self, img):
        return self._save("eref_save_pgm", img, ())

    def save_ppm(self, img, overlay, color):
        xy = np.ascontiguousarray(np.asarray(overlay, dtype=np.int32).reshape(-1, 2))
        return self._save("eref_save_ppm", img,
                          (xy.ctypes.data_as(C.POINTER(C.c_int)), len(xy), *color))

    def default_thresholds(self, field):
        gx, gy, mag = (_f64(a) for a in field)
        h, w = mag.shape
        t = abi.EdgeThresholds()
        self._check(self.lib.eref_default_thresholds(_ptr(gx), _ptr(gy), _ptr(mag), w, h,
                                                     C.byref(t)))
        return (t.low, t.high)

    def point_vote(self, dir_x, dir_y, field, cx, cy, params):
        gx, gy, mag = (_f64(a) for a in field)
        h, w = mag.shape
        out = C.c_double()
        self._check(self.lib.eref_point_vote(C.c_double(dir_x), C.c_double(dir_y), _ptr(gx),
                                             _ptr(gy), _ptr(mag), w, h, cx, cy,
                                             C.byref(params), C.byref(out)))
        return out.value

    def search_topk(self, points, field, grid, params, k, threads=0, it_range=(0, 0),
                    backend=abi.BACKEND_PARALLEL):
        assert it_range == (0, 0), "the reference API has no slab entry point"
        pts = np.ascontiguousarray(points, dtype=np.float64)
        gx, gy, mag = (_f64(a) for a in field)
        h, w = mag.shape
        out = (abi.ScoredPose * max(k, 1))()
        n = C.c_int()
        self._check(self.lib.eref_search_topk(
            pts.ctypes.data_as(C.POINTER(abi.EdgePoint)), len(pts), _ptr(gx), _ptr(gy),
            _ptr(mag), w, h, C.byref(grid), C.byref(params), backend, threads, k, out,
            C.byref(n)))
        return list(out[: n.value])

    def exhaustive_search(self, points, field, grid, params, threads=0,
                          backend=abi.BACKEND_PARALLEL):
        pts = np.ascontiguousarray(points, dtype=np.float64)
        gx, gy, mag = (_f64(a) for a in field)
        h, w = mag.shape
        out = abi.ScoredPose()
        self._check(self.lib.eref_exhaustive_search(
            pts.ctypes.data_as(C.POINTER(abi.EdgePoint)), len(pts), _ptr(gx), _ptr(gy),
            _ptr(mag), w, h, C.byref(grid), C.byref(params), backend, threads, C.byref(out)))
        return out

    def score_map(self, points, field, grid, params, max_cells):
        pts = np.ascontiguousarray(points, dtype=np.float64)
        gx, gy, mag = (_f64(a) for a in field)
        h, w = mag.shape
        total = 1
        try:
            total = int(np.prod(self.grid_counts(grid)))
        except Exception:
            pass
        out = np.zeros(max(min(total, max_cells), 1))
        self._check(self.lib.eref_score_map(pts.ctypes.data_as(C.POINTER(abi.EdgePoint)),
                                            len(pts), _ptr(gx), _ptr(gy), _ptr(mag), w, h,
                                            C.byref(grid), C.byref(params),
                                            C.c_uint64(max_cells), _ptr(out)))
        return out[:total]

    @staticmethod
    def _pyr_args(pyr):
        L = len(pyr)
        arrs = [_f64(a) for a in pyr]
        ptrs = (_dp * L)(*[_ptr(a) for a in arrs])
        dims = (C.c_int * (2 * L))()
        for l, a in enumerate(arrs):
            dims[2 * l], dims[2 * l + 1] = a.shape[1], a.shape[0]
        return arrs, ptrs, dims, L

    def prepare_levels(self, tmpl_pyr, work_pyr, cfg):
        ta, tp, td, tl = self._pyr_args(tmpl_pyr)
        wa, wp, wd, wl = self._pyr_args(work_pyr)
        h = C.c_void_p()
        self._check(self.lib.eref_prepare_levels(tp, td, tl, wp, wd, wl, C.byref(cfg),
                                                 C.byref(h)))
        try:
            models, fields = [], []
            for l in range(cfg.num_levels):
                tw, th_ = tmpl_pyr[l].shape[1], tmpl_pyr[l].shape[0]
                cap = tw * th_
                pts = np.zeros((max(cap, 1), 5))
                n, cx, cy = C.c_int(), C.c_double(), C.c_double()
                self._check(self.lib.eref_levels_model(
                    h, l, pts.ctypes.data_as(C.POINTER(abi.EdgePoint)), cap, C.byref(n),
                    C.byref(cx), C.byref(cy)))
                models.append(EdgeModel(pts[: n.value].copy(), cx.value, cy.value, l))
                ww, wh = work_pyr[l].shape[1], work_pyr[l].shape[0]
                gx, gy, mag = (np.zeros((wh, ww)) for _ in range(3))
                self._check(self.lib.eref_levels_field(h, l, _ptr(gx), _ptr(gy), _ptr(mag)))
                fields.append((gx, gy, mag))
            return models, fields
        finally:
            self.lib.eref_levels_free(h)

    def coarse_to_fine(self, tmpl_pyr, work_pyr, cfg, threads=None):
        ta, tp, td, tl = self._pyr_args(tmpl_pyr)
        wa, wp, wd, wl = self._pyr_args(work_pyr)
        out = abi.Outcome()
        self._check(self.lib.eref_coarse_to_fine(tp, td, tl, wp, wd, wl, C.byref(cfg),
                                                 C.byref(out)))
        return out

    def search_levels_timed(self, tmpl_pyr, work_pyr, cfg):
        """prepare_levels (untimed) then search_levels timed with a wall clock."""
        import time
        ta, tp, td, tl = self._pyr_args(tmpl_pyr)
        wa, wp, wd, wl = self._pyr_args(work_pyr)
        h = C.c_void_p()
        self._check(self.lib.eref_prepare_levels(tp, td, tl, wp, wd, wl, C.byref(cfg),
                                                 C.byref(h)))
        try:
            out = abi.Outcome()
            t0 = time.perf_counter()
            self._check(self.lib.eref_search_levels(h, C.byref(cfg), C.byref(out)))
            return out, time.perf_counter() - t0
        finally:
            self.lib.eref_levels_free(h)
