"""Python mirror of the reference registration API.

Same names, argument meaning and error behaviour as
/root/reference/proj/include/loopkit/registration.hpp (and the grid /
line-process entry points the path uses), implemented over the C ABI of
include/loopkit_b200.h -- the hot path runs in the sm_100a kernels of
paper_1801_01572_b200/csrc, never in Python.

  register_global        registration.hpp:121-124
  prepare_registration   registration.hpp:105-107
  run_hypotheses         registration.hpp:116-118
  evaluate_hypothesis    registration.hpp:60-63
  build_eval_grid        registration.hpp:79
  build_grid             grid.hpp:58   (SearchGrid over a target cloud)
  edge_info              line_process.hpp:15-16
  feature_nn_cache       grid.hpp:72-74
"""
from __future__ import annotations

import ctypes as C
import math
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import abi
from .errors import NoCorrespondences, check


# --------------------------------------------------------------------- types
@dataclass
class RegistrationParams:
    """registration.hpp:17-32"""

    leaf: float = 0.05
    normal_radius: float = 0.1
    feature_radius: float = 0.25
    hypothesis_count: int = 4_000_000
    similarity_tau: float = 0.9
    d_max: float = 0.075
    min_inlier_ratio: float = 0.25
    max_fitness: Optional[float] = None  # None -> d_max^2 / 2
    normal_angle_max: float = 30.0 * math.pi / 180.0
    seed: int = 0
    threads: int = 0
    device: int = -1
    # GPUs of one call (include/loopkit_b200.h lk_reg_params.device_count):
    # 0/1 = `device` alone, G = G devices from it, -1 = all visible
    device_count: int = 0

    def resolved_max_fitness(self) -> float:
        return self.max_fitness if self.max_fitness is not None else self.d_max * self.d_max / 2.0

    def to_c(self) -> abi.lk_reg_params:
        if self.device_count not in (0, 1):
            abi.prefer_process_nccl()  # G > 1 devices: NCCL inside the call
        return abi.lk_reg_params(
            leaf=self.leaf, normal_radius=self.normal_radius, feature_radius=self.feature_radius,
            hypothesis_count=int(self.hypothesis_count), similarity_tau=self.similarity_tau, d_max=self.d_max,
            min_inlier_ratio=self.min_inlier_ratio,
            max_fitness=-1.0 if self.max_fitness is None else float(self.max_fitness),
            normal_angle_max=self.normal_angle_max, seed=int(self.seed) & 0xFFFFFFFFFFFFFFFF,
            threads=int(self.threads), device=int(self.device), device_count=int(self.device_count))


@dataclass
class RigidTransform:
    """geometry.hpp:20-38: x -> rotation @ x + translation."""

    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    translation: np.ndarray = field(default_factory=lambda: np.zeros(3))

    @staticmethod
    def identity() -> "RigidTransform":
        return RigidTransform()

    def matrix(self) -> np.ndarray:
        m = np.eye(4)
        m[:3, :3] = self.rotation
        m[:3, 3] = self.translation
        return m

    @staticmethod
    def from_matrix(m) -> "RigidTransform":
        m = np.asarray(m, dtype=np.float64)
        return RigidTransform(m[:3, :3].copy(), m[:3, 3].copy())

    def packed(self) -> np.ndarray:
        """12 doubles: row-major R then t (the ABI's candidate layout)."""
        return np.concatenate([np.asarray(self.rotation, np.float64).reshape(9),
                               np.asarray(self.translation, np.float64).reshape(3)])


@dataclass
class PointCloud:
    """geometry.hpp:92-99: positions (n, 3) and optional parallel normals."""

    positions: np.ndarray
    normals: Optional[np.ndarray] = None

    def __post_init__(self):
        self.positions = np.ascontiguousarray(np.asarray(self.positions, dtype=np.float64).reshape(-1, 3))
        if self.normals is not None:
            self.normals = np.ascontiguousarray(np.asarray(self.normals, dtype=np.float64).reshape(-1, 3))
            # lk_cloud has one count for both arrays: validate_cloud's size rule
            # (geometry.cpp:93-96) is enforced before any pointer crosses the ABI
            if self.normals.shape[0] not in (0, self.positions.shape[0]):
                from .errors import MissingNormals
                raise MissingNormals("normals array must be empty or match positions")

    def size(self) -> int:
        return int(self.positions.shape[0])

    def __len__(self) -> int:
        return self.size()

    def empty(self) -> bool:
        return self.size() == 0

    def has_normals(self) -> bool:
        return self.normals is not None and self.normals.shape[0] > 0

    def pointers(self):
        """(xyz address, normals address or 0, n), cached while the arrays are
        the same objects (numpy's ctypes.data costs microseconds per call)."""
        pos, nrm = self.positions, self.normals
        cache = self.__dict__.get("_ptr_cache")
        if cache is None or cache[0] is not pos or cache[1] is not nrm:
            m = pos.shape[0]
            cache = (pos, nrm, (pos.ctypes.data if m else 0,
                                nrm.ctypes.data if nrm is not None and nrm.shape[0] > 0 else 0, m))
            self.__dict__["_ptr_cache"] = cache
        return cache[2]

    def as_c(self) -> abi.lk_cloud:
        nrm = self.normals if self.has_normals() else None
        return abi.lk_cloud(
            xyz=self.positions.ctypes.data_as(abi.dptr) if self.size() else None,
            nxyz=nrm.ctypes.data_as(abi.dptr) if nrm is not None else None,
            n=self.size())


@dataclass
class RegistrationResult:
    """registration.hpp:34-39 (+ the inlier count)."""

    transform: RigidTransform
    inlier_ratio: float
    fitness: float
    hypothesis_index: int
    inliers: int = 0


@dataclass
class HypothesisStats:
    """registration.hpp:91-99 (+ work counters: W_ref and executed evaluations)."""

    sampled: int = 0
    prerejected: int = 0
    degenerate: int = 0
    evaluated: int = 0
    qualified: int = 0
    w_ref: int = 0
    evals_executed: int = 0
    prepare_seconds: float = 0.0
    hypothesis_seconds: float = 0.0

    def _fill(self, s: abi.lk_hyp_stats) -> None:
        for name, _ in abi.lk_hyp_stats._fields_:
            setattr(self, name, getattr(s, name))


def _result(r: abi.lk_reg_result) -> Optional[RegistrationResult]:
    if not r.found:
        return None
    R = np.array(r.R[:], dtype=np.float64).reshape(3, 3)
    t = np.array(r.t[:], dtype=np.float64)
    return RegistrationResult(RigidTransform(R, t), r.inlier_ratio, r.fitness, r.hypothesis_index, r.inliers)


# --------------------------------------------------------------- context
class RegistrationContext:
    """registration.hpp:82-89: everything register_global precomputes, resident
    on one B200 (downsampled clouds, match cache, EvalGrid)."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        ns, nt = C.c_int64(), C.c_int64()
        check(abi.lib().lk_reg_ctx_sizes(self._h, C.byref(ns), C.byref(nt)))
        self.n_source, self.n_target = ns.value, nt.value
        self._cache_host = None

    @property
    def handle(self):
        return self._h

    def close(self) -> None:
        if self._h:
            abi.lib().lk_reg_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_stream(self, stream_handle: int) -> None:
        check(abi.lib().lk_reg_ctx_set_stream(self._h, C.c_void_p(stream_handle)))

    def set_profiling(self, enable: bool) -> None:
        check(abi.lib().lk_reg_ctx_set_profiling(self._h, 1 if enable else 0))

    def kernel_times(self, reset: bool = False):
        """({'k_hyp_sample': ms, 'k_kabsch': ms, 'k_score': ms}, runs) accumulated
        from CUDA events on the launch stream while profiling is enabled."""
        ms = (C.c_double * 3)()
        runs = C.c_int64()
        check(abi.lib().lk_reg_ctx_kernel_times(self._h, ms, C.byref(runs), 1 if reset else 0))
        return dict(zip(("k_hyp_sample", "k_kabsch", "k_score"), ms[:])), runs.value

    _PHASES = ("k_hyp_sample", "k_kabsch", "prep", "score_a", "score_b", "score_tail")

    def phase_times(self, reset: bool = False):
        """({kernel: ms}, runs) accumulated from CUDA events on the launch
        stream: k_hyp_sample, k_kabsch and the scorer (k_score_units +
        k_score_cta, reported as k_score_cta)."""
        ms = (C.c_double * len(self._PHASES))()
        runs = C.c_int64()
        check(abi.lib().lk_reg_ctx_phase_times(self._h, ms, len(self._PHASES), C.byref(runs), 1 if reset else 0))
        t = dict(zip(self._PHASES, ms[:]))
        return {"k_hyp_sample": t["k_hyp_sample"], "k_kabsch": t["k_kabsch"],
                "k_score_cta": t["prep"] + t["score_a"] + t["score_b"] + t["score_tail"]}, runs.value

    def attach_comm(self, unique_id: bytes, nranks: int, rank: int) -> None:
        """One process per GPU: join the NCCL communicator of `unique_id`
        (lk_nccl_unique_id on rank 0, broadcast by the caller); run_hypotheses
        then runs this rank's share and merges over NCCL."""
        abi.prefer_process_nccl()
        buf = (C.c_uint8 * 128).from_buffer_copy(bytes(unique_id))
        check(abi.lib().lk_reg_ctx_attach_comm(self._h, buf, int(nranks), int(rank)))

    def run_exchange(self, params: "RegistrationParams", records_dev_ptr: int) -> None:
        """This rank's share + the NCCL record exchange, asynchronous on the
        context stream; leaves nranks lk_reg_records at records_dev_ptr."""
        p = params.to_c()
        check(abi.lib().lk_reg_run_exchange(self._h, C.byref(p), C.c_void_p(records_dev_ptr)))

    def topology(self):
        """(devices of this context, nranks, rank)"""
        a, b, c = C.c_int32(), C.c_int32(), C.c_int32()
        check(abi.lib().lk_reg_ctx_topology(self._h, C.byref(a), C.byref(b), C.byref(c)))
        return a.value, b.value, c.value

    def download(self):
        """(source, target, cache, source_features, target_features) on the host."""
        ns, nt = self.n_source, self.n_target
        sp, sn = np.empty((ns, 3)), np.empty((ns, 3))
        tp, tn = np.empty((nt, 3)), np.empty((nt, 3))
        cache = np.empty(ns, np.int32)
        sf, tf = np.zeros((ns, 33), np.float32), np.zeros((nt, 33), np.float32)
        check(abi.lib().lk_reg_ctx_download(
            self._h, sp.ctypes.data_as(abi.dptr), sn.ctypes.data_as(abi.dptr), tp.ctypes.data_as(abi.dptr),
            tn.ctypes.data_as(abi.dptr), cache.ctypes.data_as(abi.i32ptr), sf.ctypes.data_as(abi.fptr),
            tf.ctypes.data_as(abi.fptr)))
        return PointCloud(sp, sn), PointCloud(tp, tn), cache, sf, tf

    @property
    def source(self) -> PointCloud:
        return self.download()[0]

    @property
    def target(self) -> PointCloud:
        return self.download()[1]

    @property
    def cache(self) -> np.ndarray:
        return self.download()[2]


def nccl_unique_id() -> bytes:
    """128-byte NCCL unique id for RegistrationContext.attach_comm (rank 0)."""
    abi.prefer_process_nccl()
    buf = (C.c_uint8 * 128)()
    check(abi.lib().lk_nccl_unique_id(buf))
    return bytes(buf)


def prepare_registration(source_cloud: PointCloud, target_cloud: PointCloud,
                         params: RegistrationParams) -> RegistrationContext:
    """registration.cpp:223-251. Raises TooFewPoints / MissingData."""
    s, t, p = source_cloud.as_c(), target_cloud.as_c(), params.to_c()
    h = C.c_void_p()
    check(abi.lib().lk_reg_prepare(C.byref(s), C.byref(t), C.byref(p), C.byref(h)))
    return RegistrationContext(h.value)


def registration_context(source: PointCloud, target: PointCloud, cache, params: RegistrationParams
                         ) -> RegistrationContext:
    """A RegistrationContext filled by the caller (downsampled clouds with
    normals and the feature match cache); the EvalGrid is built on device."""
    cache = np.ascontiguousarray(np.asarray(cache, dtype=np.int32))
    s, t, p = source.as_c(), target.as_c(), params.to_c()
    h = C.c_void_p()
    check(abi.lib().lk_reg_ctx_create(C.byref(s), C.byref(t), cache.ctypes.data_as(abi.i32ptr), C.byref(p),
                                      C.byref(h)))
    return RegistrationContext(h.value)


def run_hypotheses(ctx: RegistrationContext, params: RegistrationParams,
                   stats: Optional[HypothesisStats] = None) -> Optional[RegistrationResult]:
    """registration.cpp:253-332: None when no hypothesis qualifies."""
    p = params.to_c()
    r = abi.lk_reg_result()
    s = abi.lk_hyp_stats()
    if stats is not None:
        s.prepare_seconds = stats.prepare_seconds
    check(abi.lib().lk_reg_run_hypotheses(ctx.handle, C.byref(p), C.byref(r), C.byref(s)),
          allow=(abi.LK_OK, abi.LK_NO_ALIGNMENT))
    if stats is not None:
        stats._fill(s)
    return _result(r)


def run_hypotheses_range(ctx: RegistrationContext, params: RegistrationParams, begin: int, end: int,
                         device_record_ptr: Optional[int] = None) -> Optional[abi.lk_reg_record]:
    """One shard [begin, end) of the hypothesis range. With a device pointer
    the record is written there asynchronously (e.g. the rank's slot of an
    NCCL buffer); otherwise it is returned on the host."""
    p = params.to_c()
    if device_record_ptr is not None:
        check(abi.lib().lk_reg_run_range(ctx.handle, C.byref(p), int(begin), int(end),
                                         C.c_void_p(device_record_ptr), 1))
        return None
    rec = abi.lk_reg_record()
    check(abi.lib().lk_reg_run_range(ctx.handle, C.byref(p), int(begin), int(end), C.cast(C.byref(rec), C.c_void_p),
                                     0))
    return rec


def merge_records(records: Sequence[abi.lk_reg_record], n_source: int,
                  stats: Optional[HypothesisStats] = None) -> Optional[RegistrationResult]:
    """Exact merge of per-rank records under the run_hypotheses total order."""
    arr = (abi.lk_reg_record * len(records))(*records)
    r = abi.lk_reg_result()
    s = abi.lk_hyp_stats()
    check(abi.lib().lk_reg_merge_records(arr, len(records), int(n_source), C.byref(r), C.byref(s)),
          allow=(abi.LK_OK, abi.LK_NO_ALIGNMENT))
    if stats is not None:
        stats._fill(s)
    return _result(r)


def records_from_bytes(buf: np.ndarray) -> List[abi.lk_reg_record]:
    """Decode a [G x 192 B] buffer (e.g. an all-gathered NCCL buffer)."""
    raw = np.ascontiguousarray(buf).view(np.uint8).reshape(-1, C.sizeof(abi.lk_reg_record))
    return [abi.lk_reg_record.from_buffer_copy(row.tobytes()) for row in raw]


def register_global(source_cloud: PointCloud, target_cloud: PointCloud, params: RegistrationParams,
                    stats: Optional[HypothesisStats] = None) -> Optional[RegistrationResult]:
    """registration.cpp:334-343: prepare_registration + run_hypotheses."""
    s, t, p = source_cloud.as_c(), target_cloud.as_c(), params.to_c()
    r = abi.lk_reg_result()
    st = abi.lk_hyp_stats()
    check(abi.lib().lk_register_global(C.byref(s), C.byref(t), C.byref(p), C.byref(r), C.byref(st)),
          allow=(abi.LK_OK, abi.LK_NO_ALIGNMENT))
    if stats is not None:
        stats._fill(st)
    return _result(r)


# ------------------------------------------------------------------ grids
class DeviceGrid:
    """A target grid resident on the device (kind 0 EvalGrid / kind 1 SearchGrid)."""

    kind = -1

    def __init__(self, handle: int, has_normals: bool):
        self._h = C.c_void_p(handle)
        self.has_normals = has_normals
        o = (C.c_double * 3)()
        cell = C.c_double()
        dims = (C.c_int32 * 3)()
        nc, npnt = C.c_int64(), C.c_int64()
        check(abi.lib().lk_grid_dims(self._h, o, C.byref(cell), dims, C.byref(nc), C.byref(npnt)))
        self.origin = np.array(o[:])
        self.cell = cell.value
        self.dims = tuple(dims[:])
        self.ncells, self.npoints = nc.value, npnt.value

    @property
    def handle(self):
        return self._h

    def close(self):
        if self._h:
            abi.lib().lk_grid_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def download(self):
        start = np.empty(self.ncells + 1, np.int32)
        index = np.empty(self.npoints, np.int32)
        sp = np.empty((self.npoints, 3))
        sn = np.empty((self.npoints, 3))
        near = np.empty(self.ncells, np.uint8)
        check(abi.lib().lk_grid_download(self._h, start.ctypes.data_as(abi.i32ptr), index.ctypes.data_as(abi.i32ptr),
                                         sp.ctypes.data_as(abi.dptr), sn.ctypes.data_as(abi.dptr),
                                         near.ctypes.data_as(abi.u8ptr)))
        return dict(start=start, index=index, slot_position=sp, slot_normal=sn, near_occupied=near)


class EvalGrid(DeviceGrid):
    """registration.hpp:68-77"""

    kind = 0


class SearchGrid(DeviceGrid):
    """grid.hpp:21-56 semantics (cells floor(p / cell_length), exact nn_within)."""

    kind = 1


def _build(cls, cloud: PointCloud, cell: float, d_max: float, device: int):
    c = cloud.as_c()
    h = C.c_void_p()
    check(abi.lib().lk_grid_build(C.byref(c), cls.kind, float(cell), float(d_max), int(device), C.byref(h)))
    return cls(h.value, cloud.has_normals())


def build_eval_grid(target: PointCloud, d_max: float, device: int = -1) -> EvalGrid:
    """registration.cpp:80-148, built on the device."""
    return _build(EvalGrid, target, d_max, d_max, device)


def build_grid(cloud: PointCloud, cell_length: float, d_max: Optional[float] = None,
               device: int = -1) -> SearchGrid:
    """grid.cpp:32-66 cell convention; `d_max` fixes the scan radius
    ceil(d_max / cell_length) used by nn_within (defaults to cell_length)."""
    return _build(SearchGrid, cloud, cell_length, cell_length if d_max is None else d_max, device)


def _packed(transforms) -> np.ndarray:
    if isinstance(transforms, RigidTransform):
        transforms = [transforms]
    if isinstance(transforms, (list, tuple)):
        arr = np.stack([t.packed() if isinstance(t, RigidTransform) else np.asarray(t, np.float64).reshape(-1)[:12]
                        for t in transforms]) if transforms else np.zeros((0, 12))
    else:
        arr = np.asarray(transforms, np.float64)
        if arr.ndim == 3 and arr.shape[1:] == (4, 4):
            arr = np.concatenate([arr[:, :3, :3].reshape(-1, 9), arr[:, :3, 3]], axis=1)
        arr = arr.reshape(-1, 12)
    return np.ascontiguousarray(arr, dtype=np.float64)


@dataclass
class CandidateScores:
    inlier_ratio: np.ndarray
    fitness: np.ndarray
    inliers: np.ndarray  # -1 where the candidate exited on the miss budget
    best: Optional[RegistrationResult]
    qualified: int


def score_candidates(grid: DeviceGrid, source: PointCloud, transforms, params: RegistrationParams,
                     early_exit: bool = False) -> CandidateScores:
    """Explicit SE(3) candidate list: evaluate_hypothesis per candidate
    (registration.cpp:53-78 over a SearchGrid; registration.cpp:155-219 over
    an EvalGrid), plus run_hypotheses' qualification and total order."""
    rt = _packed(transforms)
    n = rt.shape[0]
    s, p = source.as_c(), params.to_c()
    per = (abi.lk_cand_score * max(n, 1))()
    best = abi.lk_reg_result()
    q = C.c_int64()
    check(abi.lib().lk_score_candidates(grid.handle, C.byref(s), rt.ctypes.data_as(abi.dptr), n, C.byref(p),
                                        1 if early_exit else 0, per, C.byref(best), C.byref(q)))
    arr = np.frombuffer(per, dtype=np.dtype([("r", "f8"), ("f", "f8"), ("i", "i8")]), count=n)
    return CandidateScores(arr["r"].copy(), arr["f"].copy(), arr["i"].copy(), _result(best), q.value)


def evaluate_hypothesis(t: RigidTransform, source: PointCloud, target: PointCloud, target_grid: SearchGrid,
                        params: RegistrationParams) -> Tuple[float, float]:
    """registration.cpp:53-78: exact (inlier_ratio, fitness) of one candidate."""
    from .errors import EmptyCloud, MissingNormals
    if source.empty() or target.empty():
        raise EmptyCloud("evaluate_hypothesis: empty cloud")
    if not source.has_normals() or not target.has_normals():
        raise MissingNormals("evaluate_hypothesis: both clouds need normals")
    sc = score_candidates(target_grid, source, [t], params)
    return float(sc.inlier_ratio[0]), float(sc.fitness[0])


# ----------------------------------------------------------- verification
@dataclass
class EdgeInfo:
    """pose_graph.hpp EdgeInfo: 6x6 information and correspondence count."""

    info: np.ndarray = field(default_factory=lambda: np.zeros((6, 6)))
    pair_count: int = 0


def edge_info_batched(clouds_i: Sequence[PointCloud], clouds_j: Sequence[PointCloud],
                      t_i: Sequence[RigidTransform], t_j: Sequence[RigidTransform], epsilon: float,
                      device: int = -1) -> List[EdgeInfo]:
    """line_process.cpp:11-33 for a batch of loop pairs (config E); pairs
    without correspondences come back with pair_count 0."""
    n = len(clouds_i)
    ci = (abi.lk_cloud * max(n, 1))(*[c.as_c() for c in clouds_i])
    cj = (abi.lk_cloud * max(n, 1))(*[c.as_c() for c in clouds_j])
    ti = np.ascontiguousarray(np.stack([t.packed() for t in t_i]) if n else np.zeros((1, 12)))
    tj = np.ascontiguousarray(np.stack([t.packed() for t in t_j]) if n else np.zeros((1, 12)))
    info = np.zeros((max(n, 1), 36))
    cnt = np.zeros(max(n, 1), np.int64)
    check(abi.lib().lk_edge_info_batched(ci, cj, ti.ctypes.data_as(abi.dptr), tj.ctypes.data_as(abi.dptr), n,
                                         float(epsilon), int(device), info.ctypes.data_as(abi.dptr),
                                         cnt.ctypes.data_as(abi.i64ptr)))
    return [EdgeInfo(info[k].reshape(6, 6).copy(), int(cnt[k])) for k in range(n)]


def edge_info(cloud_i: PointCloud, cloud_j: PointCloud, t_i: RigidTransform, t_j: RigidTransform,
              epsilon: float) -> EdgeInfo:
    """line_process.cpp:11-33. Raises EmptyCloud / NoCorrespondences."""
    e = edge_info_batched([cloud_i], [cloud_j], [t_i], [t_j], epsilon)[0]
    if e.pair_count == 0:
        raise NoCorrespondences("edge_info: no points within epsilon")
    return e


# ------------------------------------------------------- batched verification (north-star item 5)
@dataclass
class VerifyParams:
    """Config E: edge_info radius, propose_loops overlap radius,
    evaluate_hypothesis d_max / normal gate / SearchGrid cell."""

    epsilon: float = 0.05
    overlap_radius: float = 0.1
    d_max: float = 0.075
    grid_cell: float = 0.0  # <= 0 -> d_max
    normal_angle_max: float = 30.0 * math.pi / 180.0
    device: int = -1
    device_count: int = 0  # G > 1: the pairs split over G devices from `device`; -1 = all visible


@dataclass
class VerifyResult:
    info: EdgeInfo            # edge_info(Q, P, T_i, T_j, epsilon); pair_count 0 = NoCorrespondences
    overlap_hits: int         # propose_loops: posed later points within overlap_radius
    overlap: float
    inliers: int              # evaluate_hypothesis(T, P, Q)
    inlier_ratio: float
    fitness: float


def verify_batch(earlier: Sequence[PointCloud], later: Sequence[PointCloud], pose_earlier: Sequence[RigidTransform],
                 pose_later: Sequence[RigidTransform], measurement: Sequence[RigidTransform],
                 params: Optional[VerifyParams] = None) -> List[VerifyResult]:
    """Loop verification of a batch of pairs in one device pass (include/loopkit_b200.h lk_verify_batch)."""
    p = params or VerifyParams()
    n = len(earlier)
    ci, cj = _cloud_table(earlier), _cloud_table(later)
    ti, tj, tm = _pack_transforms(pose_earlier), _pack_transforms(pose_later), _pack_transforms(measurement)
    cp = abi.lk_verify_params(epsilon=float(p.epsilon), overlap_radius=float(p.overlap_radius), d_max=float(p.d_max),
                              grid_cell=float(p.grid_cell), normal_angle_max=float(p.normal_angle_max),
                              device=int(p.device), device_count=int(p.device_count))
    out = (abi.lk_verify_result * max(n, 1))()
    check(abi.lib().lk_verify_batch(ci.ctypes.data_as(C.POINTER(abi.lk_cloud)),
                                    cj.ctypes.data_as(C.POINTER(abi.lk_cloud)), ti.ctypes.data_as(abi.dptr),
                                    tj.ctypes.data_as(abi.dptr), tm.ctypes.data_as(abi.dptr), n, C.byref(cp), out))
    r = np.ctypeslib.as_array(out)[:n]
    info = np.array(r["info"]).reshape(-1, 6, 6)
    cols = [r[f].tolist() for f in ("pair_count", "overlap_hits", "overlap", "inliers", "inlier_ratio", "fitness")]
    return [VerifyResult(EdgeInfo(info[k], pc), oh, ov, il, ir, ft)
            for k, (pc, oh, ov, il, ir, ft) in enumerate(zip(*cols))]


@dataclass
class LoopParams:
    """fragments.hpp LoopParams."""

    overlap_radius: float = 0.1  # point-to-point distance counted as overlap
    min_overlap: float = 0.2     # fraction of the source fragment's points
    device: int = -1


@dataclass
class LoopProposal:
    i: int  # later fragment
    j: int  # earlier fragment
    overlap: float


def propose_loops(fragments: Sequence[PointCloud], poses: Sequence[RigidTransform],
                  loops: Sequence[Tuple[int, int]] = (), params: Optional[LoopParams] = None) -> List[LoopProposal]:
    """fragments.cpp:61-109 on the device: fragments = Fragment::cloud (local
    frame), poses = PoseGraph::poses, loops = the (i, j) of PoseGraph::loops.
    Raises MissingData when the counts differ (fragments.cpp:64-66), EmptyCloud
    for an empty fragment."""
    from .errors import MissingData
    p = params or LoopParams()
    n = len(fragments)
    if len(poses) != n:
        raise MissingData("propose_loops: one graph pose per fragment required")
    tab = _cloud_table(fragments)
    tp = _pack_transforms(poses)
    lp = np.ascontiguousarray(np.asarray(list(loops), dtype=np.int32).reshape(-1, 2)) if len(loops) else \
        np.zeros((1, 2), np.int32)
    cp = abi.lk_loop_params(overlap_radius=float(p.overlap_radius), min_overlap=float(p.min_overlap),
                            device=int(p.device), _pad=0)
    cap = max(n * n, 1)
    out = (abi.lk_loop_proposal * cap)()
    cnt = C.c_int64()
    check(abi.lib().lk_propose_loops(tab.ctypes.data_as(C.POINTER(abi.lk_cloud)), tp.ctypes.data_as(abi.dptr), n,
                                     lp.ctypes.data_as(abi.i32ptr), len(loops), C.byref(cp), out, cap,
                                     C.byref(cnt)))
    return [LoopProposal(int(out[k].i), int(out[k].j), float(out[k].overlap)) for k in range(cnt.value)]


def _pack_transforms(ts) -> np.ndarray:
    """(n, 12) row-major R then t per transform (RigidTransform.packed, batched)."""
    if not len(ts):
        return np.zeros((1, 12))
    out = np.empty((len(ts), 12))
    out[:, :9] = np.array([t.rotation for t in ts], dtype=np.float64).reshape(-1, 9)
    out[:, 9:] = np.array([t.translation for t in ts], dtype=np.float64).reshape(-1, 3)
    return out


def _cloud_table(clouds) -> np.ndarray:
    """lk_cloud[] as an (n, 3) int64 table (xyz, nxyz, n): one array instead
    of a ctypes object per cloud."""
    if not len(clouds):
        return np.zeros((1, 3), dtype=np.int64)
    return np.array([c.pointers() for c in clouds], dtype=np.int64)


# ------------------------------------------------------- ICP (north-star item 4)
@dataclass
class IcpParams:
    """Point-to-plane ICP (no reference: SPEC.md:332; spec in DESIGN.md "ICP")."""

    max_correspondence_distance: float = 0.05
    max_iterations: int = 30
    convergence_eps: float = 1e-10
    device: int = -1


@dataclass
class IcpResult:
    transform: RigidTransform
    iterations: int
    converged: bool
    correspondences: int
    rmse: float
    fitness: float
    history: np.ndarray  # (iterations evaluated, 3): correspondences, rmse, |delta|^2


def icp_point_to_plane(source: PointCloud, target: PointCloud, init: RigidTransform,
                       params: Optional[IcpParams] = None) -> IcpResult:
    """Refines `init` (source -> target) by point-to-plane ICP on the device.
    Raises EmptyCloud / MissingNormals / NoCorrespondences."""
    p = params or IcpParams()
    cp = abi.lk_icp_params(max_correspondence_distance=float(p.max_correspondence_distance),
                           max_iterations=int(p.max_iterations), device=int(p.device),
                           convergence_eps=float(p.convergence_eps))
    res = abi.lk_icp_result()
    T0 = np.ascontiguousarray(init.packed())
    hist = np.zeros((max(int(p.max_iterations), 1), 3))
    s, t = source.as_c(), target.as_c()
    check(abi.lib().lk_icp_point_to_plane(C.byref(s), C.byref(t), T0.ctypes.data_as(abi.dptr), C.byref(cp),
                                          C.byref(res), hist.ctypes.data_as(abi.dptr)))
    evaluated = min(int(res.iterations) + (0 if res.converged else 1), int(p.max_iterations))
    return IcpResult(RigidTransform(np.array(res.R[:]).reshape(3, 3), np.array(res.t[:])), int(res.iterations),
                     bool(res.converged), int(res.correspondences), float(res.rmse), float(res.fitness),
                     hist[:evaluated].copy())


# ------------------------------------------------------- prepare helpers
def feature_nn_cache(source_features: np.ndarray, target_features: np.ndarray, device: int = -1) -> np.ndarray:
    """grid.cpp:176-213 semantics pinned to the FP64 exhaustive matcher (reference.hpp:56-76)."""
    sf = np.ascontiguousarray(source_features, np.float32).reshape(-1, 33)
    tf = np.ascontiguousarray(target_features, np.float32).reshape(-1, 33)
    out = np.empty(sf.shape[0], np.int32)
    check(abi.lib().lk_feature_nn_cache(sf.ctypes.data_as(abi.fptr), sf.shape[0], tf.ctypes.data_as(abi.fptr),
                                        tf.shape[0], int(device), out.ctypes.data_as(abi.i32ptr)))
    return out


def voxel_downsample(cloud: PointCloud, leaf: float) -> PointCloud:
    """preprocess.cpp:14-59"""
    c = cloud.as_c()
    n = cloud.size()
    out = np.empty((max(n, 1), 3))
    outn = np.empty((max(n, 1), 3))
    cnt = C.c_int64()
    check(abi.lib().lk_voxel_downsample(C.byref(c), float(leaf), out.ctypes.data_as(abi.dptr),
                                        outn.ctypes.data_as(abi.dptr), C.byref(cnt)))
    k = cnt.value
    return PointCloud(out[:k].copy(), outn[:k].copy() if cloud.has_normals() else None)


def estimate_normals(cloud: PointCloud, radius: float, viewpoint=(0.0, 0.0, 0.0), device: int = -1) -> PointCloud:
    """preprocess.cpp:61-96 on the device: the cloud with normals oriented toward
    `viewpoint` (zero where fewer than 3 points lie within `radius`)."""
    c = cloud.as_c()
    out = np.zeros((max(cloud.size(), 1), 3))
    v = np.ascontiguousarray(np.asarray(viewpoint, np.float64).reshape(3))
    check(abi.lib().lk_estimate_normals(C.byref(c), float(radius), v.ctypes.data_as(abi.dptr), int(device),
                                        out.ctypes.data_as(abi.dptr)))
    return PointCloud(cloud.positions.copy(), out[:cloud.size()].copy())


def compute_fpfh(cloud: PointCloud, radius: float, threads: int = 0) -> np.ndarray:
    """fpfh.cpp:57-141"""
    c = cloud.as_c()
    out = np.zeros((cloud.size(), 33), np.float32)
    check(abi.lib().lk_compute_fpfh(C.byref(c), float(radius), int(threads), out.ctypes.data_as(abi.fptr)))
    return out


def device_count() -> int:
    return int(abi.lib().lk_device_count())
