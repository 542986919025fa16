"""ctypes mirror of the plain-data structs in include/edgealign_b200.h.

Field order and widths must match the header exactly; tests/test_abi.py checks
sizes and offsets against the compiled library.
"""
import ctypes as C
import math

EA_OK = 0
EA_ERR_INVALID_ARGUMENT = 1
EA_ERR_SIZE = 2
EA_ERR_EMPTY_MODEL = 3
EA_ERR_BOUNDS = 4
EA_ERR_BUDGET = 5
EA_ERR_GEOMETRY = 6
EA_ERR_PARSE = 7
EA_ERR_CUDA = 8
EA_ERR_INTERNAL = 9
EA_ERR_NCCL = 10
EA_COMM_ID_BYTES = 128

POLARITY_SIGNED = 0
POLARITY_IGNORE = 1
BACKEND_SERIAL = 0
BACKEND_PARALLEL = 1
BACKEND_CUDA = 2

TEMPLATE_IDS = {"rectangle": 0, "ring": 1, "l_bracket": 2, "cross": 3}
EA_MAX_LEVELS = 16

K_PI = 3.14159265358979323846  # pose.h:21


def deg_to_rad(deg):
    """pose.h:23 -- deg * (kPi / 180.0), same evaluation order."""
    return deg * (K_PI / 180.0)


def rad_to_deg(rad):
    """pose.h:24"""
    return rad * (180.0 / K_PI)


class Pose(C.Structure):
    _fields_ = [("ux", C.c_double), ("uy", C.c_double), ("theta", C.c_double)]

    def __repr__(self):
        return f"Pose(ux={self.ux!r}, uy={self.uy!r}, theta={self.theta!r})"

    def astuple(self):
        return (self.ux, self.uy, self.theta)


class PoseGrid(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("x0", "x1", "dx", "y0", "y1", "dy", "t0", "t1", "dt")]

    def __init__(self, x0=0.0, x1=0.0, dx=1.0, y0=0.0, y1=0.0, dy=1.0, t0=0.0, t1=0.0, dt=1.0):
        super().__init__(float(x0), float(x1), float(dx), float(y0), float(y1), float(dy),
                         float(t0), float(t1), float(dt))

    def __repr__(self):
        return "PoseGrid(" + ", ".join(f"{n}={getattr(self, n)!r}" for n, _ in self._fields_) + ")"


class GridCounts(C.Structure):
    _fields_ = [("nx", C.c_uint64), ("ny", C.c_uint64), ("nt", C.c_uint64)]


class ScoreParams(C.Structure):
    _fields_ = [("neighborhood", C.c_int32), ("polarity", C.c_int32), ("eps_mag", C.c_double)]

    def __init__(self, neighborhood=3, polarity=POLARITY_SIGNED, eps_mag=1e-9):
        super().__init__(int(neighborhood), int(polarity), float(eps_mag))


class EdgeThresholds(C.Structure):
    _fields_ = [("low", C.c_double), ("high", C.c_double)]


class EdgePoint(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("x_rel", "y_rel", "dx", "dy", "mag")]


class ScoredPose(C.Structure):
    _fields_ = [("score", C.c_double), ("grid_index", C.c_uint64), ("pose", Pose)]

    def __repr__(self):
        return f"ScoredPose(score={self.score!r}, grid_index={self.grid_index}, pose={self.pose!r})"


class LevelTrace(C.Structure):
    _fields_ = [("level", C.c_int32), ("_pad", C.c_int32), ("pose", Pose), ("score", C.c_double)]


class Outcome(C.Structure):
    """SearchOutcome + Detection (search.h:42-47,62-65)."""
    _fields_ = [("found", C.c_int32), ("n_trace", C.c_int32), ("pose", Pose),
                ("score", C.c_double), ("grid_index", C.c_uint64),
                ("trace", LevelTrace * EA_MAX_LEVELS)]

    def level_trace(self):
        return [(t.level, t.pose.astuple(), t.score) for t in self.trace[: self.n_trace]]

    def key(self):
        """Everything parity compares, as plain Python values."""
        return (bool(self.found), self.pose.astuple(), self.score, int(self.grid_index),
                tuple(self.level_trace()))


class SearchConfig(C.Structure):
    _fields_ = [("grid", PoseGrid), ("num_levels", C.c_int32), ("has_thresholds", C.c_int32),
                ("score_params", ScoreParams), ("thresholds", EdgeThresholds),
                ("min_score", C.c_double), ("topk", C.c_int32), ("refine_radius", C.c_int32),
                ("backend_kind", C.c_int32), ("worker_count", C.c_int32)]

    def __init__(self, grid=None, num_levels=3, score_params=None, thresholds=None,
                 min_score=0.5, topk=5, refine_radius=2, backend_kind=BACKEND_CUDA,
                 worker_count=0):
        super().__init__()
        self.grid = grid if grid is not None else PoseGrid()
        self.num_levels = num_levels
        self.score_params = score_params if score_params is not None else ScoreParams()
        if thresholds is not None:
            self.has_thresholds = 1
            self.thresholds = EdgeThresholds(*thresholds)
        self.min_score = min_score
        self.topk = topk
        self.refine_radius = refine_radius
        self.backend_kind = backend_kind
        self.worker_count = worker_count


class Stamp(C.Structure):
    """ea_stamp: one template of a multi-stamp scene (ea_compose_multi)."""
    _fields_ = [("template_id", C.c_int32), ("template_size", C.c_int32), ("pose", Pose)]

    def __init__(self, template_id="rectangle", template_size=0, pose=(0.0, 0.0, 0.0)):
        super().__init__()
        self.template_id = TEMPLATE_IDS[template_id] if isinstance(template_id, str) else template_id
        self.template_size = template_size
        self.pose = Pose(*pose)


class SceneSpec(C.Structure):
    """edgealign::SceneSpec (synth.h:67-79); theta in radians."""
    _fields_ = [("canvas_width", C.c_int32), ("canvas_height", C.c_int32),
                ("template_id", C.c_int32), ("template_size", C.c_int32),
                ("true_pose", Pose), ("clutter_segments", C.c_int32),
                ("has_occluder", C.c_int32), ("clutter_seed", C.c_uint64),
                ("occ_x", C.c_int32), ("occ_y", C.c_int32), ("occ_w", C.c_int32),
                ("occ_h", C.c_int32), ("occ_fill", C.c_double), ("gain", C.c_double),
                ("bias", C.c_double), ("gamma", C.c_double), ("noise_sigma", C.c_double),
                ("noise_seed", C.c_uint64)]

    def __init__(self, canvas_width=0, canvas_height=0, template_id="rectangle",
                 template_size=0, true_pose=(0.0, 0.0, 0.0), clutter_segments=0,
                 clutter_seed=0, occluder=None, illumination=(1.0, 0.0, 1.0),
                 noise_sigma=0.0, noise_seed=0):
        super().__init__()
        self.canvas_width = canvas_width
        self.canvas_height = canvas_height
        self.template_id = TEMPLATE_IDS[template_id] if isinstance(template_id, str) else template_id
        self.template_size = template_size
        self.true_pose = Pose(*true_pose)
        self.clutter_segments = clutter_segments
        self.clutter_seed = clutter_seed
        if occluder is not None:
            self.has_occluder = 1
            self.occ_x, self.occ_y, self.occ_w, self.occ_h, self.occ_fill = occluder
        self.gain, self.bias, self.gamma = illumination
        self.noise_sigma = noise_sigma
        self.noise_seed = noise_seed


class SearchStats(C.Structure):
    _fields_ = [("poses", C.c_uint64), ("pose_points", C.c_uint64), ("candidates", C.c_uint64),
                ("candidates_needed", C.c_uint64), ("screen_delta", C.c_double),
                ("threshold", C.c_double), ("screen_path", C.c_int32),
                ("flagged_points", C.c_int32), ("kernels_launched", C.c_int32),
                ("_pad", C.c_int32), ("screen_ms", C.c_double), ("top_ms", C.c_double),
                ("image_ms", C.c_double), ("refine_ms", C.c_double)]


def isfinite_grid(g):
    return all(math.isfinite(getattr(g, n)) for n, _ in PoseGrid._fields_)


class CommId(C.Structure):
    """ea_comm_id: an ncclUniqueId, created on rank 0 and handed out of band."""
    _fields_ = [("internal", C.c_char * EA_COMM_ID_BYTES)]


def comm_id_bytes(cid):
    """The 128 raw bytes of an ea_comm_id (c_char arrays stop at NUL; this does not)."""
    return C.string_at(C.addressof(cid), EA_COMM_ID_BYTES)


def comm_id_from_bytes(raw):
    cid = CommId()
    C.memmove(C.addressof(cid), bytes(raw), EA_COMM_ID_BYTES)
    return cid


class WorkItem(C.Structure):
    """ea_work_item: one (model, theta slab) of a multi-model sharded search."""
    _fields_ = [("rank", C.c_int32), ("model", C.c_int32), ("it_begin", C.c_uint64),
                ("it_end", C.c_uint64), ("cost", C.c_double)]

    def astuple(self):
        return (self.rank, self.model, self.it_begin, self.it_end, self.cost)
