"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of the CPU oracle (lk_oracle.h).

The oracle restates the reference's registration path on the CPU
(/root/reference/proj/src/registration.cpp and friends). Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
import this module; the product never does.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from dataclasses import dataclass
from typing import Optional, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "liblk_oracle.so")

dptr = C.POINTER(C.c_double)
fptr = C.POINTER(C.c_float)
i32ptr = C.POINTER(C.c_int32)
i64ptr = C.POINTER(C.c_int64)
u8ptr = C.POINTER(C.c_uint8)
u32ptr = C.POINTER(C.c_uint32)
u64ptr = C.POINTER(C.c_uint64)


class or_params(C.Structure):
    _fields_ = [
        ("leaf", C.c_double), ("normal_radius", C.c_double), ("feature_radius", C.c_double),
        ("hypothesis_count", C.c_int64), ("similarity_tau", C.c_double), ("d_max", C.c_double),
        ("min_inlier_ratio", C.c_double), ("max_fitness", C.c_double), ("normal_angle_max", C.c_double),
        ("seed", C.c_uint64), ("threads", C.c_int32), ("device_count", C.c_int32),
    ]


class or_result(C.Structure):
    _fields_ = [
        ("R", C.c_double * 9), ("t", C.c_double * 3), ("inlier_ratio", C.c_double), ("fitness", C.c_double),
        ("inliers", C.c_int64), ("hypothesis_index", C.c_int64), ("found", C.c_int32), ("_pad", C.c_int32),
    ]


class or_stats(C.Structure):
    _fields_ = [
        ("sampled", C.c_int64), ("prerejected", C.c_int64), ("degenerate", C.c_int64), ("evaluated", C.c_int64),
        ("qualified", C.c_int64), ("w_ref", C.c_int64), ("near_occupied", C.c_int64),
        ("slots_scanned", C.c_int64), ("nn_hits", C.c_int64), ("prepare_seconds", C.c_double),
        ("hypothesis_seconds", C.c_double),
    ]


_SIGS = {
    "or_last_error": (C.c_char_p, []),
    "or_splitmix64": (C.c_uint64, [C.c_uint64]),
    "or_rng_u64": (None, [C.c_uint64, C.c_uint64, C.c_int64, u64ptr]),
    "or_rng_bounded": (None, [C.c_uint64, C.c_uint64, C.c_uint32, C.c_int64, u32ptr]),
    "or_rng_double": (None, [C.c_uint64, C.c_uint64, C.c_int64, dptr]),
    "or_sample_quadruples": (C.c_int, [C.c_int32, i32ptr, C.c_int64, C.c_uint64, C.c_uint64, C.c_int32, i32ptr,
                                       i32ptr]),
    "or_prerejected": (C.c_int, [dptr, dptr, C.c_double]),
    "or_kabsch": (C.c_int, [dptr, dptr, C.c_int64, dptr, dptr, dptr]),
    "or_svd3": (C.c_int, [dptr, dptr, dptr, dptr]),
    "or_search_grid_build": (C.c_void_p, [dptr, C.c_int64, C.c_double, dptr, C.POINTER(C.c_int)]),
    "or_search_grid_free": (None, [C.c_void_p]),
    "or_nn_within": (C.c_int, [C.c_void_p, dptr, C.c_double, i32ptr, dptr]),
    "or_nn_nearest": (C.c_int, [C.c_void_p, dptr, i32ptr, dptr]),
    "or_radius_search": (C.c_int64, [C.c_void_p, dptr, C.c_double, i32ptr, C.c_int64]),
    "or_bf_nn_within": (C.c_int, [dptr, C.c_int64, dptr, C.c_double, i32ptr, dptr]),
    "or_eval_grid_build": (C.c_void_p, [dptr, dptr, C.c_int64, C.c_double, C.POINTER(C.c_int)]),
    "or_eval_grid_free": (None, [C.c_void_p]),
    "or_eval_grid_dims": (None, [C.c_void_p, dptr, dptr, i32ptr, i64ptr, i64ptr]),
    "or_eval_grid_arrays": (None, [C.c_void_p, i32ptr, i32ptr, dptr, dptr, u8ptr]),
    "or_evaluate_against_grid": (C.c_int, [C.c_void_p, dptr, dptr, C.c_int64, dptr, dptr, C.c_double, C.c_double,
                                           C.c_int64, dptr, dptr, i64ptr, i64ptr]),
    "or_evaluate_hypothesis": (C.c_int, [dptr, dptr, dptr, dptr, C.c_int64, dptr, dptr, C.c_int64, C.c_double,
                                         C.POINTER(or_params), dptr, dptr, i64ptr]),
    "or_score_candidates": (C.c_int, [dptr, dptr, C.c_int64, dptr, dptr, C.c_int64, dptr, C.c_int64, C.c_int32,
                                      C.c_int32, C.c_double, C.POINTER(or_params), dptr, dptr, i64ptr, i32ptr,
                                      C.POINTER(or_result), i64ptr]),
    "or_voxel_downsample": (C.c_int, [dptr, dptr, C.c_int64, C.c_double, dptr, dptr, i64ptr]),
    "or_estimate_normals": (C.c_int, [dptr, C.c_int64, C.c_double, dptr, C.c_int32, dptr]),
    "or_compute_fpfh": (C.c_int, [dptr, dptr, C.c_int64, C.c_double, C.c_int32, fptr]),
    "or_feature_nn_cache": (C.c_int, [fptr, C.c_int64, fptr, C.c_int64, C.c_int32, i32ptr]),
    "or_prepare": (C.c_void_p, [dptr, dptr, C.c_int64, dptr, dptr, C.c_int64, C.POINTER(or_params),
                                C.POINTER(C.c_int)]),
    "or_ctx_from_prepared": (C.c_void_p, [dptr, dptr, C.c_int64, dptr, dptr, C.c_int64, i32ptr, C.c_double,
                                          C.POINTER(C.c_int)]),
    "or_ctx_sizes": (None, [C.c_void_p, i64ptr, i64ptr]),
    "or_ctx_get": (None, [C.c_void_p, dptr, dptr, dptr, dptr, i32ptr, fptr, fptr]),
    "or_ctx_free": (None, [C.c_void_p]),
    "or_run_hypotheses": (C.c_int, [C.c_void_p, C.POINTER(or_params), C.c_int64, C.c_int64, C.POINTER(or_result),
                                    C.POINTER(or_stats)]),
    "or_better": (C.c_int, [C.POINTER(or_result), C.POINTER(or_result)]),
    "or_edge_info": (C.c_int, [dptr, C.c_int64, dptr, C.c_int64, dptr, dptr, dptr, dptr, C.c_double, dptr, i64ptr]),
}

_lib = None


def build() -> str:
    """Compile the oracle (make -C oracle). Returns the library path."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(status: int) -> None:
    if status != 0:
        m = lib().or_last_error()
        raise OracleError(status, m.decode() if m else "")


def _d(a) -> Optional[np.ndarray]:
    if a is None:
        return None
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def _p(a):
    return None if a is None else a.ctypes.data_as(dptr)


def params(hypothesis_count=4_000_000, seed=0, d_max=0.075, leaf=0.05, normal_radius=0.1, feature_radius=0.25,
           similarity_tau=0.9, min_inlier_ratio=0.25, max_fitness=None, normal_angle_max=30.0 * math.pi / 180.0,
           threads=0) -> or_params:
    return or_params(leaf=leaf, normal_radius=normal_radius, feature_radius=feature_radius,
                     hypothesis_count=int(hypothesis_count), similarity_tau=similarity_tau, d_max=d_max,
                     min_inlier_ratio=min_inlier_ratio, max_fitness=-1.0 if max_fitness is None else max_fitness,
                     normal_angle_max=normal_angle_max, seed=int(seed), threads=threads, device_count=0)


def params_from(p) -> or_params:
    """or_params from a paper_1801_01572_b200.RegistrationParams (same fields)."""
    return params(hypothesis_count=p.hypothesis_count, seed=p.seed, d_max=p.d_max, leaf=p.leaf,
                  normal_radius=p.normal_radius, feature_radius=p.feature_radius, similarity_tau=p.similarity_tau,
                  min_inlier_ratio=p.min_inlier_ratio, max_fitness=p.max_fitness,
                  normal_angle_max=p.normal_angle_max, threads=p.threads)


@dataclass
class Result:
    found: bool
    R: np.ndarray
    t: np.ndarray
    inlier_ratio: float
    fitness: float
    inliers: int
    hypothesis_index: int


def _result(r: or_result) -> Result:
    return Result(bool(r.found), np.array(r.R[:]).reshape(3, 3), np.array(r.t[:]), r.inlier_ratio, r.fitness,
                  r.inliers, r.hypothesis_index)


def rng_u64(seed, stream, n):
    out = np.empty(n, np.uint64)
    lib().or_rng_u64(seed, stream, n, out.ctypes.data_as(u64ptr))
    return out


def rng_bounded(seed, stream, bound, n):
    out = np.empty(n, np.uint32)
    lib().or_rng_bounded(seed, stream, bound, n, out.ctypes.data_as(u32ptr))
    return out


def sample_quadruples(source_size, cache, seed, stream, trials):
    cache = np.ascontiguousarray(cache, np.int32)
    s = np.empty((trials, 4), np.int32)
    t = np.empty((trials, 4), np.int32)
    _check(lib().or_sample_quadruples(source_size, cache.ctypes.data_as(i32ptr), cache.size, seed, stream, trials,
                                      s.ctypes.data_as(i32ptr), t.ctypes.data_as(i32ptr)))
    return s, t


def prerejected(src4, dst4, tau) -> bool:
    s, d = _d(src4), _d(dst4)
    return bool(lib().or_prerejected(_p(s), _p(d), tau))


def kabsch(src, dst) -> Tuple[np.ndarray, np.ndarray]:
    s, d = _d(src), _d(dst)
    R, t, sg = np.empty(9), np.empty(3), np.empty(3)
    _check(lib().or_kabsch(_p(s), _p(d), s.shape[0], _p(R), _p(t), _p(sg)))
    return R.reshape(3, 3), t


def svd3(A):
    A = _d(A)
    U, S, V = np.empty(9), np.empty(3), np.empty(9)
    _check(lib().or_svd3(_p(A), _p(U), _p(S), _p(V)))
    return U.reshape(3, 3), S, V.reshape(3, 3)


class SearchGrid:
    def __init__(self, xyz, cell, center=(0.0, 0.0, 0.0)):
        self.xyz = _d(xyz)
        c = _d(center)
        st = C.c_int()
        self.h = lib().or_search_grid_build(_p(self.xyz), self.xyz.shape[0], cell, _p(c), C.byref(st))
        _check(st.value)

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_search_grid_free(self.h)

    def nn_within(self, q, d_max):
        q = _d(q)
        i, d = C.c_int32(), C.c_double()
        return (i.value, d.value) if lib().or_nn_within(self.h, _p(q), d_max, C.byref(i), C.byref(d)) else None

    def nn_nearest(self, q):
        q = _d(q)
        i, d = C.c_int32(), C.c_double()
        _check(lib().or_nn_nearest(self.h, _p(q), C.byref(i), C.byref(d)))
        return i.value, d.value

    def radius_search(self, q, r):
        q = _d(q)
        cap = self.xyz.shape[0]
        out = np.empty(max(cap, 1), np.int32)
        n = lib().or_radius_search(self.h, _p(q), r, out.ctypes.data_as(i32ptr), cap)
        return out[:n].tolist()


def bf_nn_within(xyz, q, d_max):
    x, q = _d(xyz), _d(q)
    i, d = C.c_int32(), C.c_double()
    return (i.value, d.value) if lib().or_bf_nn_within(_p(x), x.shape[0], _p(q), d_max, C.byref(i), C.byref(d)) \
        else None


class EvalGrid:
    def __init__(self, xyz, nrm, d_max):
        self.xyz, self.nrm = _d(xyz), _d(nrm)
        st = C.c_int()
        self.h = lib().or_eval_grid_build(_p(self.xyz), _p(self.nrm), self.xyz.shape[0], d_max, C.byref(st))
        _check(st.value)
        o, cell, dims, nc, npnt = np.empty(3), C.c_double(), (C.c_int32 * 3)(), C.c_int64(), C.c_int64()
        lib().or_eval_grid_dims(self.h, _p(o), C.byref(cell), dims, C.byref(nc), C.byref(npnt))
        self.origin, self.cell, self.dims, self.ncells, self.npoints = o, cell.value, tuple(dims[:]), nc.value, \
            npnt.value

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_eval_grid_free(self.h)

    def arrays(self):
        start = np.empty(self.ncells + 1, np.int32)
        index = np.empty(self.npoints, np.int32)
        sp, sn = np.empty((self.npoints, 3)), np.empty((self.npoints, 3))
        near = np.empty(self.ncells, np.uint8)
        lib().or_eval_grid_arrays(self.h, start.ctypes.data_as(i32ptr), index.ctypes.data_as(i32ptr), _p(sp),
                                  _p(sn), near.ctypes.data_as(u8ptr))
        return dict(start=start, index=index, slot_position=sp, slot_normal=sn, near_occupied=near)

    def evaluate(self, src_xyz, src_n, R, t, d_max, cos_max, miss_budget):
        s, n, R, t = _d(src_xyz), _d(src_n), _d(R), _d(t)
        r, f, inl, vis = C.c_double(), C.c_double(), C.c_int64(), C.c_int64()
        ok = lib().or_evaluate_against_grid(self.h, _p(s), _p(n), s.shape[0], _p(R), _p(t), d_max, cos_max,
                                            miss_budget, C.byref(r), C.byref(f), C.byref(inl), C.byref(vis))
        return bool(ok), r.value, f.value, inl.value, vis.value


def evaluate_hypothesis(R, t, src_xyz, src_n, tgt_xyz, tgt_n, grid_cell, p: or_params):
    R, t, s, sn, q, qn = _d(R), _d(t), _d(src_xyz), _d(src_n), _d(tgt_xyz), _d(tgt_n)
    r, f, inl = C.c_double(), C.c_double(), C.c_int64()
    _check(lib().or_evaluate_hypothesis(_p(R), _p(t), _p(s), _p(sn), 0 if s is None else s.shape[0], _p(q), _p(qn),
                                        0 if q is None else q.shape[0], grid_cell, C.byref(p), C.byref(r),
                                        C.byref(f), C.byref(inl)))
    return r.value, f.value, inl.value


def score_candidates(src_xyz, src_n, tgt_xyz, tgt_n, Rt, mode, early_exit, grid_cell, p: or_params):
    s, sn, q, qn, rt = _d(src_xyz), _d(src_n), _d(tgt_xyz), _d(tgt_n), _d(Rt).reshape(-1, 12)
    n = rt.shape[0]
    ratio, fit = np.empty(n), np.empty(n)
    inl = np.empty(n, np.int64)
    sc = np.empty(n, np.int32)
    best = or_result()
    qual = C.c_int64()
    _check(lib().or_score_candidates(_p(s), _p(sn), s.shape[0], _p(q), _p(qn), q.shape[0], _p(rt), n, mode,
                                     early_exit, grid_cell, C.byref(p), _p(ratio), _p(fit),
                                     inl.ctypes.data_as(i64ptr), sc.ctypes.data_as(i32ptr), C.byref(best),
                                     C.byref(qual)))
    return dict(ratio=ratio, fitness=fit, inliers=inl, scored=sc, best=_result(best), qualified=qual.value)


def voxel_downsample(xyz, nrm, leaf):
    x, n = _d(xyz), _d(nrm)
    N = x.shape[0]
    ox, on = np.empty((max(N, 1), 3)), np.empty((max(N, 1), 3))
    cnt = C.c_int64()
    _check(lib().or_voxel_downsample(_p(x), _p(n), N, leaf, _p(ox), _p(on), C.byref(cnt)))
    k = cnt.value
    return ox[:k].copy(), (on[:k].copy() if n is not None else None)


def estimate_normals(xyz, radius, viewpoint=(0.0, 0.0, 0.0), threads=0):
    """preprocess.cpp:61-96 (oracle restatement; Eigen's eigensolver restated)."""
    x = _d(xyz)
    v = _d(np.asarray(viewpoint, np.float64).reshape(1, 3))
    out = np.zeros((x.shape[0], 3))
    _check(lib().or_estimate_normals(_p(x), x.shape[0], radius, _p(v), threads, _p(out)))
    return out


def compute_fpfh(xyz, nrm, radius, threads=0):
    x, n = _d(xyz), _d(nrm)
    out = np.zeros((x.shape[0], 33), np.float32)
    _check(lib().or_compute_fpfh(_p(x), _p(n), x.shape[0], radius, threads, out.ctypes.data_as(fptr)))
    return out


def feature_nn_cache(sf, tf, threads=0):
    sf = np.ascontiguousarray(sf, np.float32).reshape(-1, 33)
    tf = np.ascontiguousarray(tf, np.float32).reshape(-1, 33)
    out = np.empty(sf.shape[0], np.int32)
    _check(lib().or_feature_nn_cache(sf.ctypes.data_as(fptr), sf.shape[0], tf.ctypes.data_as(fptr), tf.shape[0],
                                     threads, out.ctypes.data_as(i32ptr)))
    return out


class Context:
    """RegistrationContext of the oracle."""

    def __init__(self, h):
        self.h = h
        ns, nt = C.c_int64(), C.c_int64()
        lib().or_ctx_sizes(h, C.byref(ns), C.byref(nt))
        self.ns, self.nt = ns.value, nt.value

    @staticmethod
    def prepare(sxyz, sn, txyz, tn, p: or_params) -> "Context":
        s, sn, t, tn = _d(sxyz), _d(sn), _d(txyz), _d(tn)
        st = C.c_int()
        h = lib().or_prepare(_p(s), _p(sn), s.shape[0], _p(t), _p(tn), t.shape[0], C.byref(p), C.byref(st))
        _check(st.value)
        return Context(h)

    @staticmethod
    def from_prepared(sxyz, sn, txyz, tn, cache, d_max) -> "Context":
        s, sn, t, tn = _d(sxyz), _d(sn), _d(txyz), _d(tn)
        cache = np.ascontiguousarray(cache, np.int32)
        st = C.c_int()
        h = lib().or_ctx_from_prepared(_p(s), _p(sn), s.shape[0], _p(t), _p(tn), t.shape[0],
                                       cache.ctypes.data_as(i32ptr), d_max, C.byref(st))
        _check(st.value)
        return Context(h)

    def get(self):
        sp, sn = np.empty((self.ns, 3)), np.empty((self.ns, 3))
        tp, tn = np.empty((self.nt, 3)), np.empty((self.nt, 3))
        cache = np.empty(self.ns, np.int32)
        sf, tf = np.zeros((self.ns, 33), np.float32), np.zeros((self.nt, 33), np.float32)
        lib().or_ctx_get(self.h, _p(sp), _p(sn), _p(tp), _p(tn), cache.ctypes.data_as(i32ptr),
                         sf.ctypes.data_as(fptr), tf.ctypes.data_as(fptr))
        return dict(src=sp, src_n=sn, tgt=tp, tgt_n=tn, cache=cache, src_feat=sf, tgt_feat=tf)

    def run(self, p: or_params, begin=0, end=None):
        end = p.hypothesis_count if end is None else end
        r, s = or_result(), or_stats()
        _check(lib().or_run_hypotheses(self.h, C.byref(p), begin, end, C.byref(r), C.byref(s)))
        stats = {name: getattr(s, name) for name, _ in or_stats._fields_}
        return _result(r), stats

    def __del__(self):
        if getattr(self, "h", None):
            lib().or_ctx_free(self.h)


def edge_info(ci, cj, Ri, ti, Rj, tj, eps):
    a, b = _d(ci), _d(cj)
    Ri, ti, Rj, tj = _d(Ri), _d(ti), _d(Rj), _d(tj)
    info = np.empty(36)
    cnt = C.c_int64()
    _check(lib().or_edge_info(_p(a), a.shape[0], _p(b), b.shape[0], _p(Ri), _p(ti), _p(Rj), _p(tj), eps, _p(info),
                              C.byref(cnt)))
    return info.reshape(6, 6), cnt.value


class or_icp_result(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("correspondences", C.c_int64),
                ("rmse", C.c_double), ("fitness", C.c_double)]


def icp_point_to_plane(src_xyz, tgt_xyz, tgt_n, R0, t0, max_dist, max_iter=30, eps=1e-10):
    """The frozen ICP spec (lk_oracle.cpp "ICP point-to-plane"): returns
    (R, t, or_icp_result, history[max_iter, 3])."""
    L = lib()
    L.or_icp_point_to_plane.restype = C.c_int
    s, t, tn = _d(src_xyz), _d(tgt_xyz), _d(tgt_n)
    R0 = _d(np.asarray(R0).reshape(9))
    t0 = _d(np.asarray(t0).reshape(3))
    R, tt = np.empty(9), np.empty(3)
    res = or_icp_result()
    hist = np.zeros((max(int(max_iter), 1), 3))
    _check(L.or_icp_point_to_plane(_p(s), C.c_int64(len(s)), _p(t), _p(tn), C.c_int64(len(t)), _p(R0), _p(t0),
                                   C.c_double(max_dist), C.c_int32(max_iter), C.c_double(eps), _p(R), _p(tt),
                                   C.byref(res), _p(hist)))
    return R.reshape(3, 3), tt, res, hist


def overlap_hits(later, T_later_R, T_later_t, earlier, T_earlier_R, T_earlier_t, r):
    """propose_loops' overlap hit count of one pair (fragments.cpp:67-100)."""
    L = lib()
    L.or_overlap_hits.restype = C.c_int
    a, b = _d(later), _d(earlier)
    Rl, tl = _d(np.asarray(T_later_R).reshape(9)), _d(np.asarray(T_later_t).reshape(3))
    Re, te = _d(np.asarray(T_earlier_R).reshape(9)), _d(np.asarray(T_earlier_t).reshape(3))
    h = C.c_int64()
    _check(L.or_overlap_hits(_p(a), C.c_int64(len(a)), _p(Rl), _p(tl), _p(b), C.c_int64(len(b)), _p(Re), _p(te),
                             C.c_double(r), C.byref(h)))
    return h.value
