"""Python mirror of the reference `edgealign` API over the C-ABI.

Names, argument meaning and error behaviour follow
proj/include/edgealign/*.h (cited per function); arrays are numpy float64
images of shape (height, width).  Every compute call runs on the CUDA device
of a `Context`; host-only calls are the template side (edge-model extraction)
and the synthetic-scene generator.
"""
import ctypes as C
from dataclasses import dataclass, field as dc_field

import numpy as np

from . import abi
from ._lib import lib
from .abi import (BACKEND_CUDA, BACKEND_PARALLEL, BACKEND_SERIAL, POLARITY_IGNORE,
                  POLARITY_SIGNED, EdgePoint, Outcome, Pose, PoseGrid, SceneSpec,
                  ScoredPose, ScoreParams, SearchConfig, deg_to_rad, rad_to_deg)
from .errors import raise_for_status

_dp = C.POINTER(C.c_double)


def _check(st):
    if st != abi.EA_OK:
        L = lib()
        raise_for_status(st, L.ea_last_error(), L.ea_last_error_value())


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _ptr(a):
    return a.ctypes.data_as(_dp)


@dataclass
class GradientField:
    """edgealign::GradientField (gradient.h:17-36)."""
    gx: np.ndarray
    gy: np.ndarray
    mag: np.ndarray

    @property
    def width(self):
        return self.mag.shape[1]

    @property
    def height(self):
        return self.mag.shape[0]

    def __iter__(self):
        return iter((self.gx, self.gy, self.mag))


@dataclass
class EdgeModel:
    """edgealign::EdgeModel (edge_model.h:40-45): points (n, 5) =
    x_rel, y_rel, dx, dy, mag in row-major source order."""
    points: np.ndarray
    centroid_x: float = 0.0
    centroid_y: float = 0.0
    source_level: int = 0

    def __len__(self):
        return len(self.points)


def model_point_count(model):
    """edge_model.cpp:26-28"""
    return len(model.points)


class Context:
    """A CUDA device + stream + scratch arena (one host thread at a time)."""

    def __init__(self, device=0):
        h = C.c_void_p()
        _check(lib().ea_ctx_create(int(device), C.byref(h)))
        self.handle = h
        self.device = device

    def close(self):
        if self.handle:
            lib().ea_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_ptr):
        _check(lib().ea_ctx_set_stream(self.handle, C.c_void_p(stream_ptr)))

    def synchronize(self):
        _check(lib().ea_ctx_synchronize(self.handle))

    def stats(self):
        s = abi.SearchStats()
        _check(lib().ea_ctx_last_stats(self.handle, C.byref(s)))
        return {n: getattr(s, n) for n, _ in abi.SearchStats._fields_ if not n.startswith("_")}

    def set_timing(self, on=True):
        _check(lib().ea_ctx_set_timing(self.handle, 1 if on else 0))

    def kernel_launches(self):
        return int(lib().ea_ctx_kernel_launches(self.handle))

    # ---- multi-GPU (ea_comm_*): one context per GPU, one rank per context ----
    def comm_init(self, rank, world, comm_id):
        """Join this context's device to an NCCL communicator (collective)."""
        _check(lib().ea_comm_init(self.handle, int(rank), int(world), C.byref(comm_id)))

    def comm_info(self):
        r, w = C.c_int(), C.c_int()
        _check(lib().ea_comm_info(self.handle, C.byref(r), C.byref(w)))
        return r.value, w.value

    def has_comm(self):
        r, w = C.c_int(), C.c_int()
        return lib().ea_comm_info(self.handle, C.byref(r), C.byref(w)) == abi.EA_OK

    def comm_destroy(self):
        _check(lib().ea_comm_destroy(self.handle))


_default = {}


def host_array(shape, dtype=np.float64):
    """A numpy array in pinned host memory from the library (ea_host_alloc,
    cudaHostAlloc), freed with the array.  Images staged here reach the
    device at the link's full rate (B200: ~55 GB/s H2D measured, where a
    torch pin_memory() buffer measured 29-47 GB/s); detect / detect_batch
    copy them without staging."""
    import weakref
    dt = np.dtype(dtype)
    n = int(np.prod(shape)) * dt.itemsize
    p = C.c_void_p()
    _check(lib().ea_host_alloc(max(n, 1), C.byref(p)))
    raw = (C.c_char * max(n, 1)).from_address(p.value)
    weakref.finalize(raw, lib().ea_host_free, C.c_void_p(p.value))
    return np.frombuffer(raw, dtype=dt, count=int(np.prod(shape))).reshape(shape)


def default_context(device=0):
    ctx = _default.get(device)
    if ctx is None:
        ctx = _default[device] = Context(device)
    return ctx


class DeviceField:
    """A gradient field resident on the device (ea_field)."""

    def __init__(self, handle, ctx):
        self.handle, self.ctx = handle, ctx

    @classmethod
    def upload(cls, field, ctx=None):
        ctx = ctx or default_context()
        gx, gy, mag = (_f64(a) for a in field)
        h = C.c_void_p()
        _check(lib().ea_field_upload(ctx.handle, _ptr(gx), _ptr(gy), _ptr(mag), mag.shape[1],
                                     mag.shape[0], C.byref(h)))
        return cls(h, ctx)

    @classmethod
    def from_image(cls, image, ctx=None):
        ctx = ctx or default_context()
        img = _f64(image)
        h = C.c_void_p()
        _check(lib().ea_field_from_image(ctx.handle, _ptr(img), img.shape[1], img.shape[0],
                                         C.byref(h)))
        return cls(h, ctx)

    def download(self):
        w, h = C.c_int(), C.c_int()
        _check(lib().ea_field_dims(self.handle, C.byref(w), C.byref(h)))
        gx, gy, mag = (np.zeros((h.value, w.value)) for _ in range(3))
        _check(lib().ea_field_download(self.ctx.handle, self.handle, _ptr(gx), _ptr(gy),
                                       _ptr(mag)))
        return GradientField(gx, gy, mag)

    def __del__(self):
        if getattr(self, "handle", None):
            lib().ea_field_free(self.handle)
            self.handle = None


class DeviceModel:
    """An edge model resident on the device (ea_model)."""

    def __init__(self, model, ctx=None):
        ctx = ctx or default_context()
        pts = np.ascontiguousarray(model.points, dtype=np.float64).reshape(-1, 5)
        h = C.c_void_p()
        _check(lib().ea_model_create(ctx.handle, pts.ctypes.data_as(C.POINTER(EdgePoint)),
                                     len(pts), float(model.centroid_x), float(model.centroid_y),
                                     int(model.source_level), C.byref(h)))
        self.handle, self.ctx, self.n = h, ctx, len(pts)
        self._keep = pts

    def __del__(self):
        if getattr(self, "handle", None):
            lib().ea_model_free(self.handle)
            self.handle = None


def extract_edge_model_device(field, thresholds=None, level=0, ctx=None):
    """extract_edge_model (edge_model.cpp:53-149) on the device
    (ea_field_extract_model); thresholds None = default_thresholds.
    -> EdgeModel with the points read back."""
    ctx = ctx or default_context()
    f = _field(field, ctx)
    h = C.c_void_p()
    th = None if thresholds is None else C.byref(
        thresholds if isinstance(thresholds, abi.EdgeThresholds) else abi.EdgeThresholds(*thresholds))
    _check(lib().ea_field_extract_model(ctx.handle, f.handle, th, int(level), C.byref(h)))
    try:
        n, cx, cy = C.c_int(), C.c_double(), C.c_double()
        _check(lib().ea_model_points(h, None, 0, C.byref(n), C.byref(cx), C.byref(cy)))
        pts = np.zeros((max(n.value, 1), 5))
        _check(lib().ea_model_points(h, pts.ctypes.data_as(C.POINTER(EdgePoint)), n.value,
                                     C.byref(n), C.byref(cx), C.byref(cy)))
    finally:
        lib().ea_model_free(h)
    return EdgeModel(pts[: n.value], cx.value, cy.value, int(level))


def _field(f, ctx):
    return f if isinstance(f, DeviceField) else DeviceField.upload(f, ctx)


def _model(m, ctx):
    return m if isinstance(m, DeviceModel) else DeviceModel(m, ctx)


# ---- pose geometry (pose.h:45-113) ------------------------------------------------
def grid_counts(grid):
    """pose.h:52-67 -> (nx, ny, nt)"""
    c = abi.GridCounts()
    _check(lib().ea_compute_grid_counts(C.byref(grid), C.byref(c)))
    return (c.nx, c.ny, c.nt)


def grid_size(grid):
    """pose.h:69-72"""
    nx, ny, nt = grid_counts(grid)
    return nx * ny * nt


def pose_at(grid, index):
    """pose.h:77-92"""
    p = Pose()
    _check(lib().ea_pose_at(C.byref(grid), C.c_uint64(index), C.byref(p)))
    return p


# ---- image (image.cpp:248-291, gradient.cpp:12-27) --------------------------------
def max_pyramid_levels(image_or_w, h=None):
    """image.cpp:263-272"""
    if h is None:
        h, w = np.shape(image_or_w)
    else:
        w = image_or_w
    return lib().ea_max_pyramid_levels(int(w), int(h))


def downsample(image, ctx=None):
    """image.cpp:248-261 (device 2x2 box mean)."""
    ctx = ctx or default_context()
    img = _f64(image)
    h, w = img.shape
    out = np.zeros((max(h // 2, 1), max(w // 2, 1)))
    _check(lib().ea_downsample(ctx.handle, _ptr(img), w, h, _ptr(out)))
    return out


def build_pyramid(image, num_levels, ctx=None):
    """image.cpp:274-291 -> list of level images (level 0 = the input)."""
    ctx = ctx or default_context()
    img = _f64(image)
    h, w = img.shape
    dims = [(w >> l, h >> l) for l in range(max(num_levels, 1))]
    out = np.zeros(sum(a * b for a, b in dims))
    _check(lib().ea_build_pyramid(ctx.handle, _ptr(img), w, h, int(num_levels), _ptr(out)))
    res, off = [], 0
    for lw, lh in dims:
        res.append(out[off: off + lw * lh].reshape(lh, lw).copy())
        off += lw * lh
    return res


def compute_gradients(image, ctx=None):
    """gradient.cpp:12-27 (device Sobel)."""
    ctx = ctx or default_context()
    img = _f64(image)
    h, w = img.shape
    gx, gy, mag = (np.zeros((h, w)) for _ in range(3))
    _check(lib().ea_compute_gradients(ctx.handle, _ptr(img), w, h, _ptr(gx), _ptr(gy),
                                      _ptr(mag)))
    return GradientField(gx, gy, mag)


# ---- template side (edge_model.cpp:17-149) -------------------------------------
def default_thresholds(field):
    """edge_model.cpp:17-24 -> (low, high)"""
    mag = _f64(field[2] if isinstance(field, tuple) else field.mag)
    t = abi.EdgeThresholds()
    _check(lib().ea_default_thresholds(_ptr(mag), mag.shape[1], mag.shape[0], C.byref(t)))
    return (t.low, t.high)


def extract_edge_model(field, thresholds, level=0):
    """edge_model.cpp:53-149"""
    gx, gy, mag = (_f64(a) for a in field)
    h, w = mag.shape
    cap = max(w * h, 1)
    pts = np.zeros((cap, 5))
    n, cx, cy = C.c_int(), C.c_double(), C.c_double()
    th = abi.EdgeThresholds(*thresholds)
    _check(lib().ea_extract_edge_model(_ptr(gx), _ptr(gy), _ptr(mag), w, h, C.byref(th), level,
                                       pts.ctypes.data_as(C.POINTER(EdgePoint)), cap,
                                       C.byref(n), C.byref(cx), C.byref(cy)))
    return EdgeModel(pts[: n.value].copy(), cx.value, cy.value, level)


# ---- similarity (similarity.cpp:15-126) ---------------------------------------
def validate(params):
    """similarity.cpp:15-23"""
    _check(lib().ea_validate_params(C.byref(params)))


def point_vote(dir_x, dir_y, field, cx, cy, params, ctx=None):
    """similarity.cpp:58-64"""
    ctx = ctx or default_context()
    f = _field(field, ctx)
    out = C.c_double()
    _check(lib().ea_point_vote(ctx.handle, float(dir_x), float(dir_y), f.handle, int(cx),
                               int(cy), C.byref(params), C.byref(out)))
    return out.value


def rotate_model(model, theta, ctx=None):
    """similarity.cpp:68-88 -> (px, py, dx, dy)"""
    ctx = ctx or default_context()
    m = _model(model, ctx)
    n = m.n
    px, py, dx, dy = (np.zeros(n) for _ in range(4))
    _check(lib().ea_rotate_model(ctx.handle, m.handle, float(theta), _ptr(px), _ptr(py),
                                 _ptr(dx), _ptr(dy)))
    return px, py, dx, dy


def pose_score(model, pose, field, params, ctx=None):
    """similarity.cpp:121-126 -> (value, n_inbounds)"""
    ctx = ctx or default_context()
    m, f = _model(model, ctx), _field(field, ctx)
    p = pose if isinstance(pose, Pose) else Pose(*pose)
    v, n = C.c_double(), C.c_int()
    _check(lib().ea_pose_score(ctx.handle, m.handle, C.byref(p), f.handle, C.byref(params),
                               C.byref(v), C.byref(n)))
    return v.value, n.value


# ---- search (search.cpp:144-202) ----------------------------------------------------
def search_topk(model, field, grid, params, backend=BACKEND_CUDA, k=5, ctx=None):
    """search.cpp:155-167 -> [ScoredPose] by (score desc, index asc)"""
    ctx = ctx or default_context()
    m, f = _model(model, ctx), _field(field, ctx)
    out = (ScoredPose * max(int(k), 1))()
    n = C.c_int()
    _check(lib().ea_search_topk(ctx.handle, m.handle, f.handle, C.byref(grid), C.byref(params),
                                int(backend), int(k), out, C.byref(n)))
    return list(out[: n.value])


def exhaustive_search(model, field, grid, params, backend=BACKEND_CUDA, ctx=None):
    """search.cpp:144-153 -> ScoredPose (score, grid_index, pose)"""
    return search_topk(model, field, grid, params, backend, 1, ctx)[0]


def search_topk_slab(model, field, grid, params, k, it_begin, it_end, ctx=None):
    """One theta slab of run_search's partition (search.cpp:116-120)."""
    ctx = ctx or default_context()
    m, f = _model(model, ctx), _field(field, ctx)
    out = (ScoredPose * max(int(k), 1))()
    n = C.c_int()
    _check(lib().ea_search_topk_slab(ctx.handle, m.handle, f.handle, C.byref(grid),
                                     C.byref(params), int(k), C.c_uint64(it_begin),
                                     C.c_uint64(it_end), out, C.byref(n)))
    return list(out[: n.value])


def merge_topk(items, k):
    """The run_search merge (search.cpp:130-139)."""
    arr = (ScoredPose * max(len(items), 1))(*items)
    out = (ScoredPose * max(int(k), 1))()
    n = C.c_int()
    _check(lib().ea_merge_topk(arr, len(items), int(k), out, C.byref(n)))
    return list(out[: n.value])


def score_map(model, field, grid, params, max_cells, ctx=None):
    """search.cpp:169-202 (exact fp64 on the device)."""
    ctx = ctx or default_context()
    m, f = _model(model, ctx), _field(field, ctx)
    total = None
    try:
        total = grid_size(grid)
    except Exception:
        total = 1
    out = np.zeros(max(min(total, int(max_cells)), 1))
    _check(lib().ea_score_map(ctx.handle, m.handle, f.handle, C.byref(grid), C.byref(params),
                              C.c_uint64(int(max_cells)), _ptr(out)))
    return out[:total]


def screen_map(model, field, grid, params, max_cells=1 << 28, ctx=None):
    """fp32 screening scores of every pose and their error bound delta."""
    ctx = ctx or default_context()
    m, f = _model(model, ctx), _field(field, ctx)
    total = grid_size(grid)
    out = np.zeros(max(min(total, int(max_cells)), 1), dtype=np.float32)
    d = C.c_double()
    _check(lib().ea_screen_map(ctx.handle, m.handle, f.handle, C.byref(grid), C.byref(params),
                               C.c_uint64(int(max_cells)),
                               out.ctypes.data_as(C.POINTER(C.c_float)), C.byref(d)))
    return out[:total], d.value


# ---- coarse to fine (search.cpp:204-364) ------------------------------------------
def _pyr_args(pyr):
    arrs = [_f64(a) for a in pyr]
    L = len(arrs)
    ptrs = (_dp * max(L, 1))(*[_ptr(a) for a in arrs])
    dims = (C.c_int * max(2 * L, 2))()
    for l, a in enumerate(arrs):
        dims[2 * l], dims[2 * l + 1] = a.shape[1], a.shape[0]
    return arrs, ptrs, dims, L


class PyramidLevels:
    """edgealign::PyramidLevels (search.h:94-97) resident on the device."""

    def __init__(self, handle, ctx):
        self.handle, self.ctx = handle, ctx

    def __len__(self):
        return lib().ea_levels_count(self.handle)

    def model(self, level):
        lv = C.c_void_p(self.handle.value if isinstance(self.handle, C.c_void_p) else self.handle)
        n, cx, cy = C.c_int(), C.c_double(), C.c_double()
        _check(lib().ea_levels_model(lv, level, None, 0, C.byref(n), C.byref(cx), C.byref(cy)))
        pts = np.zeros((max(n.value, 1), 5))
        _check(lib().ea_levels_model(lv, level, pts.ctypes.data_as(C.POINTER(EdgePoint)), n.value,
                                     C.byref(n), C.byref(cx), C.byref(cy)))
        return EdgeModel(pts[: n.value].copy(), cx.value, cy.value, level)

    def field(self, level):
        h = lib().ea_levels_field(self.handle, level)
        if not h:
            raise IndexError(level)
        f = DeviceField(C.c_void_p(h), self.ctx)
        try:
            return f.download()
        finally:
            f.handle = None  # owned by the levels object

    def set_image(self, image):
        img = _f64(image)
        _check(lib().ea_levels_set_image(self.ctx.handle, self.handle, _ptr(img), img.shape[1],
                                         img.shape[0]))

    def __del__(self):
        if getattr(self, "handle", None):
            lib().ea_levels_free(self.handle)
            self.handle = None


def prepare_levels(template_pyr, working_pyr, config, ctx=None):
    """search.cpp:208-238"""
    ctx = ctx or default_context()
    ta, tp, td, tl = _pyr_args(template_pyr)
    wa, wp, wd, wl = _pyr_args(working_pyr)
    h = C.c_void_p()
    _check(lib().ea_prepare_levels(ctx.handle, tp, td, tl, wp, wd, wl, C.byref(config),
                                   C.byref(h)))
    return PyramidLevels(h, ctx)


def prepare_models(template, config, ctx=None):
    """Template side of prepare_levels from a level-0 template (device pyramid)."""
    ctx = ctx or default_context()
    t = _f64(template)
    h = C.c_void_p()
    _check(lib().ea_prepare_models(ctx.handle, _ptr(t), t.shape[1], t.shape[0], C.byref(config),
                                   C.byref(h)))
    return PyramidLevels(h, ctx)


def search_levels(levels, config):
    """search.cpp:254-357"""
    out = Outcome()
    _check(lib().ea_search_levels(levels.ctx.handle, levels.handle, C.byref(config),
                                  C.byref(out)))
    return out


def search_top_slab(levels, config, it_begin, it_end):
    out = (ScoredPose * max(config.topk, 1))()
    n = C.c_int()
    _check(lib().ea_search_top_slab(levels.ctx.handle, levels.handle, C.byref(config),
                                    C.c_uint64(it_begin), C.c_uint64(it_end), out, C.byref(n)))
    return list(out[: n.value])


def search_top_slab_async(levels, config, it_begin, it_end, d_rows):
    """Device-resident slab search: k rows {score, index, ux, uy, theta}
    (float64) written to the device address `d_rows` on the context's stream;
    no host sync (ea_search_top_slab_async)."""
    _check(lib().ea_search_top_slab_async(levels.ctx.handle, levels.handle, C.byref(config),
                                          C.c_uint64(it_begin), C.c_uint64(it_end),
                                          C.c_void_p(int(d_rows))))


def merge_rows_async(ctx, d_rows, n_rows, k, d_out):
    """`better` merge of n_rows device rows into k device rows (no sync)."""
    _check(lib().ea_merge_rows_async(ctx.handle, C.c_void_p(int(d_rows)), int(n_rows), int(k),
                                     C.c_void_p(int(d_out))))


def theta_slab(nt, rank, world):
    """[it_begin, it_end) of `rank`: the reference's block partition
    (search.cpp:116-120) on the theta axis (ea_theta_slab)."""
    b, e = C.c_uint64(), C.c_uint64()
    lib().ea_theta_slab(C.c_uint64(int(nt)), int(rank), int(world), C.byref(b), C.byref(e))
    return b.value, e.value


def comm_unique_id():
    """An ncclUniqueId (ea_comm_unique_id) for rank 0 to hand to every rank."""
    cid = abi.CommId()
    _check(lib().ea_comm_unique_id(C.byref(cid)))
    return cid


def gather_rows_async(ctx, d_local, k, d_merged):
    """NCCL all-gather of every rank's k device rows + device `better` merge
    into k rows at d_merged (ea_gather_rows_async; no host sync)."""
    _check(lib().ea_gather_rows_async(ctx.handle, C.c_void_p(int(d_local)), int(k),
                                      C.c_void_p(int(d_merged))))


def search_levels_sharded(levels, config):
    """search_levels sharded by theta over the context's communicator."""
    out = Outcome()
    _check(lib().ea_search_levels_sharded(levels.ctx.handle, levels.handle, C.byref(config),
                                          C.byref(out)))
    return out


def async_status(ctx, cap=4096):
    """Sync; -> (overflowed, [screen-kernel ms of the timed searches since the last call])."""
    of, n = C.c_int(), C.c_int()
    times = (C.c_float * cap)()
    _check(lib().ea_ctx_async_status(ctx.handle, C.byref(of), times, cap, C.byref(n)))
    return bool(of.value), [times[i] for i in range(n.value)]


def refine(levels, config, seeds):
    arr = (ScoredPose * max(len(seeds), 1))(*seeds)
    out = Outcome()
    _check(lib().ea_refine(levels.ctx.handle, levels.handle, C.byref(config), arr, len(seeds),
                           C.byref(out)))
    return out


def coarse_to_fine(template_pyr, working_pyr, config, ctx=None):
    """search.cpp:359-364"""
    ctx = ctx or default_context()
    ta, tp, td, tl = _pyr_args(template_pyr)
    wa, wp, wd, wl = _pyr_args(working_pyr)
    out = Outcome()
    _check(lib().ea_coarse_to_fine(ctx.handle, tp, td, tl, wp, wd, wl, C.byref(config),
                                   C.byref(out)))
    return out


class Detector:
    """Production detect: template models prepared once, then one call per
    host image (H2D + device pyramid + gradients + search_levels + D2H)."""

    def __init__(self, template, config, ctx=None):
        self.ctx = ctx or default_context()
        self.config = config
        self.levels = prepare_models(template, config, self.ctx)

    def detect(self, image):
        img = image if (isinstance(image, np.ndarray) and image.dtype == np.float64
                        and image.flags.c_contiguous) else _f64(image)
        out = Outcome()
        _check(lib().ea_detect(self.ctx.handle, self.levels.handle, _ptr(img), img.shape[1],
                               img.shape[0], C.byref(self.config), C.byref(out)))
        return out


    def detect_sharded(self, image, shape=None):
        """Theta-sharded detect over the context's communicator
        (ea_detect_sharded, collective): rank 0 passes the host image, the
        other ranks None and `shape` = (h, w).  Same outcome on every rank."""
        if image is None:
            h, w = shape
            ptr = None
        else:
            img = image if (isinstance(image, np.ndarray) and image.dtype == np.float64
                            and image.flags.c_contiguous) else _f64(image)
            h, w = img.shape
            ptr = _ptr(img)
        out = Outcome()
        _check(lib().ea_detect_sharded(self.ctx.handle, self.levels.handle, ptr, w, h,
                                       C.byref(self.config), C.byref(out)))
        return out

    def detect_batch(self, images):
        """Throughput mode: one call for many same-size host images (pinned
        buffers overlap their H2D with the previous image's search)."""
        imgs = [i if (isinstance(i, np.ndarray) and i.dtype == np.float64 and i.flags.c_contiguous)
                else _f64(i) for i in images]
        if not imgs:
            return []
        h, w = imgs[0].shape
        if any(i.shape != (h, w) for i in imgs):
            raise ValueError("detect_batch needs images of one size")
        ptrs = (_dp * len(imgs))(*[_ptr(i) for i in imgs])
        outs = (Outcome * len(imgs))()
        _check(lib().ea_detect_batch(self.ctx.handle, self.levels.handle, ptrs, len(imgs), w, h,
                                     C.byref(self.config), outs))
        return list(outs)


def detect_multi(detectors, image):
    """Multi-model detect (ea_detect_multi): one image, several Detectors that
    share a context and a config; the working pyramid is built once (into the
    first detector's levels).  -> one Outcome per detector."""
    if not detectors:
        return []
    ctx, cfg = detectors[0].ctx, detectors[0].config
    for d in detectors:
        if d.ctx is not ctx:
            raise ValueError("detect_multi needs detectors on one context")
    img = image if (isinstance(image, np.ndarray) and image.dtype == np.float64
                    and image.flags.c_contiguous) else _f64(image)
    hs = (C.c_void_p * len(detectors))(*[d.levels.handle for d in detectors])
    outs = (Outcome * len(detectors))()
    _check(lib().ea_detect_multi(ctx.handle, hs, len(detectors), _ptr(img), img.shape[1],
                                 img.shape[0], C.byref(cfg), outs))
    return list(outs)


def plan_multi(plane_poses, thetas, n_top, world, fixed_evals=6.6e7):
    """ea_plan_multi: the (model, theta slab) work items of a multi-model
    sharded search, as (rank, model, it_begin, it_end, cost) tuples."""
    n = len(n_top)
    pp = (C.c_uint64 * max(n, 1))(*[int(x) for x in plane_poses])
    th = (C.c_uint64 * max(n, 1))(*[int(x) for x in thetas])
    nt = (C.c_int * max(n, 1))(*[int(x) for x in n_top])
    cap = max(n * int(world), 1)
    items = (abi.WorkItem * cap)()
    cnt = C.c_int()
    _check(lib().ea_plan_multi(pp, th, nt, n, int(world), float(fixed_evals), items, cap,
                               C.byref(cnt)))
    return [items[i].astuple() for i in range(cnt.value)]


def gather_rows_multi_async(ctx, d_local, n_models, k, d_merged):
    """NCCL all-gather of every rank's n_models x k device rows + per-model
    `better` merge into d_merged (ea_gather_rows_multi_async; no host sync)."""
    _check(lib().ea_gather_rows_multi_async(ctx.handle, C.c_void_p(int(d_local)), int(n_models),
                                            int(k), C.c_void_p(int(d_merged))))


def detect_multi_sharded(detectors, image, shape=None):
    """Multi-model detect sharded over the first detector's communicator
    (ea_detect_multi_sharded, collective): rank 0 passes the host image, the
    other ranks None and `shape` = (h, w).  -> one Outcome per detector."""
    if not detectors:
        return []
    ctx, cfg = detectors[0].ctx, detectors[0].config
    for d in detectors:
        if d.ctx is not ctx:
            raise ValueError("detect_multi_sharded needs detectors on one context")
    if image is None:
        h, w = shape
        ptr = None
    else:
        img = image if (isinstance(image, np.ndarray) and image.dtype == np.float64
                        and image.flags.c_contiguous) else _f64(image)
        h, w = img.shape
        ptr = _ptr(img)
    hs = (C.c_void_p * len(detectors))(*[d.levels.handle for d in detectors])
    outs = (Outcome * len(detectors))()
    _check(lib().ea_detect_multi_sharded(ctx.handle, hs, len(detectors), ptr, w, h,
                                         C.byref(cfg), outs))
    return list(outs)


# ---- Netpbm codecs (image.cpp:26-219) -------------------------------------------------
def luminance_to_byte(v):
    return int(lib().ea_luminance_to_byte(float(v)))


def load_pgm(data):
    """PGM bytes (P2 / P5) -> float64 image (H, W)."""
    data = bytes(data)
    w, h = C.c_int(), C.c_int()
    _check(lib().ea_load_pgm(data, len(data), None, 0, C.byref(w), C.byref(h)))
    out = np.zeros((h.value, w.value))
    _check(lib().ea_load_pgm(data, len(data), out.ctypes.data, out.size, C.byref(w),
                             C.byref(h)))
    return out


def _netpbm(fn, img, *extra):
    img = _f64(img)
    h, w = img.shape
    n = C.c_size_t()
    _check(fn(_ptr(img), w, h, *extra, None, 0, C.byref(n)))
    out = (C.c_ubyte * n.value)()
    _check(fn(_ptr(img), w, h, *extra, out, n.value, C.byref(n)))
    return bytes(out)


def save_pgm(img):
    """float64 image -> P5 bytes (clamped, rounded half up)."""
    return _netpbm(lib().ea_save_pgm, img)


def save_ppm(img, overlay=(), color=(255, 0, 0)):
    """float64 image -> P6 bytes, gray with `overlay` (x, y) pixels in `color`."""
    xy = np.ascontiguousarray(np.asarray(overlay, dtype=np.int32).reshape(-1, 2))
    return _netpbm(lib().ea_save_ppm, img, xy.ctypes.data_as(C.POINTER(C.c_int)), len(xy),
                   *[int(c) for c in color])


def overlay_points(model, pose):
    """Pixels (n, 2) of the model's points projected at `pose` (x, y, theta)."""
    pts = np.ascontiguousarray(getattr(model, "points", model), dtype=np.float64).reshape(-1, 5)
    out = np.zeros((max(len(pts), 1), 2), dtype=np.int32)
    p = pose if isinstance(pose, Pose) else Pose(*pose)
    _check(lib().ea_overlay_points(pts.ctypes.data_as(C.POINTER(EdgePoint)), len(pts),
                                   C.byref(p), out.ctypes.data_as(C.POINTER(C.c_int))))
    return out[: len(pts)]


def detect_result_json(outcome, n_model_points, elapsed_ms, backend="cuda"):
    """DetectResult (SPEC.md cli-bench: pose (x px, y px, theta degrees),
    score, n_model_points, elapsed_ms, backend, level_trace) as a JSON text
    with exactly those keys; theta reported in degrees."""
    import json
    p = outcome.pose
    trace = [{"level": int(t.level), "x": t.pose.ux, "y": t.pose.uy,
              "theta_deg": rad_to_deg(t.pose.theta), "score": t.score}
             for t in outcome.trace[: outcome.n_trace]]
    return json.dumps({"pose": {"x": p.ux, "y": p.uy, "theta_deg": rad_to_deg(p.theta)},
                       "score": outcome.score, "n_model_points": int(n_model_points),
                       "elapsed_ms": float(elapsed_ms), "backend": backend,
                       "level_trace": trace})


def load_pgm_file(path):
    with open(path, "rb") as f:
        return load_pgm(f.read())


def save_pgm_file(img, path):
    with open(path, "wb") as f:
        f.write(save_pgm(img))


def save_ppm_file(img, path, overlay=(), color=(255, 0, 0)):
    with open(path, "wb") as f:
        f.write(save_ppm(img, overlay, color))


# ---- synthetic scenes (synth.cpp:62-300) -----------------------------------------
def render_template(template_id, size):
    tid = abi.TEMPLATE_IDS[template_id] if isinstance(template_id, str) else template_id
    out = np.zeros((max(size, 1), max(size, 1)))
    _check(lib().ea_render_template(int(tid), int(size), _ptr(out)))
    return out


def compose_multi(spec, stamps):
    """Multi-stamp scene (ea_compose_multi): spec's canvas, clutter, occluder,
    illumination and noise; `stamps` = [(template_id, size, (ux, uy, theta))]."""
    arr = (abi.Stamp * max(len(stamps), 1))(*[abi.Stamp(t, s, p) for t, s, p in stamps])
    canvas = np.zeros((max(spec.canvas_height, 1), max(spec.canvas_width, 1)))
    _check(lib().ea_compose_multi(C.byref(spec), arr, len(stamps), _ptr(canvas)))
    return canvas


def compose_scene(spec):
    """-> (scene, template_image, truth_pose, occluded_fraction)"""
    canvas = np.zeros((max(spec.canvas_height, 1), max(spec.canvas_width, 1)))
    tmpl = np.zeros((max(spec.template_size, 1), max(spec.template_size, 1)))
    pose, occ = Pose(), C.c_double()
    _check(lib().ea_compose_scene(C.byref(spec), _ptr(canvas), _ptr(tmpl), C.byref(pose),
                                  C.byref(occ)))
    return canvas, tmpl, pose.astuple(), occ.value


# ---- BenchRow CSV (SPEC.md cmd_bench, "sample,backend,workers,run,elapsed_ms") ----------
BENCH_CSV_HEADER = "sample,backend,workers,run,elapsed_ms"


def bench_rows(samples, reps=5, warmup=1, backends=("cuda",), config=None, ctx=None):
    """The reference's bench rows (SPEC.md BenchRow / cmd_bench) for this
    library: for each (name, template, image) sample, `warmup` untimed then
    `reps` timed detects per backend; only the search is timed (models are
    prepared before, I/O excluded).  The CUDA backend is the only backend of
    this library (every BackendKind runs on the device, search.h:14-20);
    a sample whose backends disagree on the pose raises (cmd_bench exit 3).
    -> list of dict rows {sample, backend, workers, run, elapsed_ms}."""
    import time
    rows = []
    for name, tmpl, img in samples:
        cfg = config or SearchConfig()
        det = Detector(tmpl, cfg, ctx)
        det.levels.set_image(img)
        poses = set()
        for backend in backends:
            kind = {"serial": BACKEND_SERIAL, "parallel": BACKEND_PARALLEL,
                    "cuda": BACKEND_CUDA}[backend]
            bcfg = SearchConfig(grid=cfg.grid, num_levels=cfg.num_levels,
                                score_params=cfg.score_params, min_score=cfg.min_score,
                                topk=cfg.topk, refine_radius=cfg.refine_radius,
                                backend_kind=kind, worker_count=cfg.worker_count)
            for run in range(warmup + reps):
                t0 = time.perf_counter()
                out = search_levels(det.levels, bcfg)
                ms = (time.perf_counter() - t0) * 1e3
                if run >= warmup:
                    rows.append({"sample": name, "backend": backend,
                                 "workers": int(cfg.worker_count), "run": run - warmup,
                                 "elapsed_ms": ms})
            poses.add(out.key()[:2])  # found + pose
        if len(poses) > 1:
            raise Error(f"backends disagree on the pose of sample {name}")
    return rows


def bench_csv(rows):
    """BenchRow CSV text with the reference's exact header."""
    lines = [BENCH_CSV_HEADER]
    for r in rows:
        if not r["elapsed_ms"] > 0:
            raise ValueError("BenchRow invariant: elapsed_ms > 0")
        name = str(r["sample"])
        if any(c in name for c in ',"\n'):
            name = '"' + name.replace('"', '""') + '"'
        lines.append(f"{name},{r['backend']},{int(r['workers'])},{int(r['run'])},"
                     f"{float(r['elapsed_ms']):.6f}")
    return "\n".join(lines) + "\n"
