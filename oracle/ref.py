"""TEST INFRASTRUCTURE ONLY: ctypes wrapper of oracle/_ref/liblk_ref.so -- the
REFERENCE's own registration code (/root/reference/proj/src/*.cpp, compiled
unmodified against oracle/ref_shim/ by oracle/Makefile.ref; C ABI in
oracle/ref_capi.cpp).

Used by tests/ to pin the oracle restatement (oracle.py) and, through the
golden files it generates (tests/golden/make_ref_golden.py), the device path
to the reference's own code; bench.py's reference arm times it. The product
never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

import oracle as O
from oracle import dptr, fptr, i32ptr, i64ptr, u8ptr, or_params, or_result, or_stats

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "liblk_ref.so")
TESTS_PATH = os.path.join(HERE, "_ref", "ref_unit_tests")
REF_SRC = "/root/reference/proj"

_SIGS = {
    "rf_last_error": (C.c_char_p, []),
    "rf_max_threads": (C.c_int, []),
    "rf_registration_pair": (C.c_void_p, [C.c_uint64, C.c_double, C.POINTER(C.c_int)]),
    "rf_negative_pair": (C.c_void_p, [C.c_uint64, C.c_double, C.POINTER(C.c_int)]),
    "rf_frame_pair": (C.c_void_p, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                   C.c_double, C.c_int, C.c_double, C.c_int, C.c_int, C.c_int,
                                   C.POINTER(C.c_int)]),
    "rf_submap_pair": (C.c_void_p, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                    C.c_int, C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "rf_surface_pair": (C.c_void_p, [C.c_uint64, C.c_double, C.c_double, C.POINTER(C.c_int)]),
    "rf_random_cloud": (C.c_void_p, [C.c_uint64, C.c_uint64, C.c_int, C.c_double, C.c_double, C.c_int,
                                     C.POINTER(C.c_int)]),
    "rf_count": (C.c_int64, [C.c_void_p, C.c_int]),
    "rf_has_normals": (C.c_int, [C.c_void_p, C.c_int]),
    "rf_get": (None, [C.c_void_p, C.c_int, dptr, dptr]),
    "rf_truth": (None, [C.c_void_p, dptr, dptr, dptr]),
    "rf_free": (None, [C.c_void_p]),
    "rf_random_transform": (None, [C.c_uint64, C.c_uint64, C.c_int, C.c_double, C.c_double, dptr, dptr]),
    "rf_transform_from_twist": (None, [dptr, dptr, dptr]),
    "rf_compose": (None, [dptr, dptr, dptr, dptr, dptr, dptr]),
    "rf_inverse": (None, [dptr, dptr, dptr, dptr]),
    "rf_apply": (None, [dptr, dptr, dptr, C.c_int64, dptr]),
    "rf_kabsch": (C.c_int, [dptr, dptr, C.c_int64, dptr, dptr]),
    "rf_svd3": (None, [dptr, dptr, dptr, dptr]),
    "rf_voxel_downsample": (C.c_int, [dptr, dptr, C.c_int64, C.c_double, dptr, dptr, i64ptr]),
    "rf_estimate_normals": (C.c_int, [dptr, C.c_int64, C.c_double, dptr, C.c_int32, dptr]),
    "rf_compute_fpfh": (C.c_int, [dptr, dptr, C.c_int64, C.c_double, C.c_int32, fptr]),
    "rf_feature_nn_cache": (C.c_int, [fptr, C.c_int64, fptr, C.c_int64, C.c_int32, C.c_int32, i32ptr]),
    "rf_prepare": (C.c_void_p, [dptr, dptr, C.c_int64, dptr, dptr, C.c_int64, C.POINTER(or_params),
                                C.POINTER(C.c_int)]),
    "rf_ctx_from_prepared": (C.c_void_p, [dptr, dptr, C.c_int64, dptr, dptr, C.c_int64, i32ptr, C.c_double,
                                          C.POINTER(C.c_int)]),
    "rf_ctx_sizes": (None, [C.c_void_p, i64ptr, i64ptr]),
    "rf_ctx_get": (None, [C.c_void_p, dptr, dptr, dptr, dptr, i32ptr, fptr, fptr]),
    "rf_ctx_eval_dims": (None, [C.c_void_p, dptr, dptr, i32ptr, i64ptr]),
    "rf_ctx_eval_arrays": (None, [C.c_void_p, i32ptr, i32ptr, dptr, dptr, u8ptr]),
    "rf_ctx_free": (None, [C.c_void_p]),
    "rf_run_hypotheses": (C.c_int, [C.c_void_p, C.POINTER(or_params), C.POINTER(or_result), C.POINTER(or_stats)]),
    "rf_register_global": (C.c_int, [dptr, dptr, C.c_int64, dptr, dptr, C.c_int64, C.POINTER(or_params),
                                      C.POINTER(or_result), C.POINTER(or_stats)]),
    "rf_evaluate_hypothesis": (C.c_int, [dptr, dptr, dptr, dptr, C.c_int64, dptr, dptr, C.c_int64, C.c_double,
                                         C.POINTER(or_params), dptr, dptr]),
    "rf_nn_within_batch": (C.c_int, [dptr, C.c_int64, C.c_double, dptr, C.c_int64, C.c_double, i32ptr, dptr]),
    "rf_edge_info": (C.c_int, [dptr, C.c_int64, dptr, C.c_int64, dptr, dptr, dptr, dptr, C.c_double, dptr,
                               i64ptr]),
    "rf_edge_residual": (C.c_double, [dptr, dptr, dptr, dptr, dptr, dptr, dptr, C.c_int64, C.POINTER(C.c_int)]),
    "rf_update_weight": (C.c_double, [C.c_double, C.c_double]),
    "rf_propose_loops": (C.c_int64, [dptr, i64ptr, C.c_int32, dptr, dptr, i32ptr, C.c_int32, C.c_double,
                                     C.c_double, i32ptr, i32ptr, dptr, C.c_int64]),
}

_lib = None


def available() -> bool:
    """True when oracle/_ref/liblk_ref.so exists (built from /root/reference) or can be built here."""
    return os.path.exists(LIB_PATH) or os.path.isdir(REF_SRC)


def build() -> str:
    """make -f Makefile.ref (needs /root/reference; the GPU box uses the prebuilt files)."""
    subprocess.run(["make", "-s", "-j8", "-C", HERE, "-f", "Makefile.ref"], check=True)
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


class RefError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _check(status: int) -> None:
    if status != 0:
        m = lib().rf_last_error()
        raise RefError(status, m.decode() if m else "")


_d, _p = O._d, O._p


def _fixture(h, st) -> dict:
    _check(st.value)
    L = lib()
    try:
        out = {}
        for w, name in ((0, "source"), (1, "target")):
            n = L.rf_count(h, w)
            if n < 0:
                continue
            xyz = np.empty((n, 3))
            nrm = np.empty((n, 3)) if L.rf_has_normals(h, w) else None
            L.rf_get(h, w, _p(xyz), _p(nrm))
            out[name] = (xyz, nrm)
        R, t, sc = np.empty(9), np.empty(3), C.c_double()
        L.rf_truth(h, _p(R), _p(t), C.byref(sc))
        out["truth"] = (R.reshape(3, 3), t)
        out["scalar"] = sc.value
        return out
    finally:
        L.rf_free(h)


def registration_pair(seed, leaf=0.05):
    st = C.c_int()
    return _fixture(lib().rf_registration_pair(seed, leaf, C.byref(st)), st)


def negative_pair(seed, leaf=0.05):
    st = C.c_int()
    return _fixture(lib().rf_negative_pair(seed, leaf, C.byref(st)), st)


def frame_pair(seed=1, boxes=6, width=640, height=480, fx=525.0, fy=525.0, cx=319.5, cy=239.5, stride=1,
               noise=0.005, frames=90, frame_a=0, frame_b=6):
    st = C.c_int()
    return _fixture(lib().rf_frame_pair(seed, boxes, width, height, fx, fy, cx, cy, stride, noise, frames, frame_a,
                                        frame_b, C.byref(st)), st)


def submap_pair(seed=2, boxes=6, views=8, width=640, height=480, stride=1, noise=0.005, frames=90, a0=0, b0=8,
                step=2):
    st = C.c_int()
    return _fixture(lib().rf_submap_pair(seed, boxes, views, width, height, stride, noise, frames, a0, b0, step,
                                         C.byref(st)), st)


def surface_pair(seed=1, density=1000.0, noise=0.005):
    st = C.c_int()
    return _fixture(lib().rf_surface_pair(seed, density, noise, C.byref(st)), st)


def random_cloud(n, seed, stream=0, lo=-1.0, hi=1.0, with_normals=False):
    st = C.c_int()
    return _fixture(lib().rf_random_cloud(seed, stream, n, lo, hi, 1 if with_normals else 0, C.byref(st)), st)


def random_transform(seed, stream=0, max_angle=np.pi * 0.9, max_trans=1.0, skip_draws=0):
    R, t = np.empty(9), np.empty(3)
    lib().rf_random_transform(seed, stream, skip_draws, max_angle, max_trans, _p(R), _p(t))
    return R.reshape(3, 3), t


def transform_from_twist(xi):
    x = _d(np.asarray(xi, np.float64).reshape(6))
    R, t = np.empty(9), np.empty(3)
    lib().rf_transform_from_twist(_p(x), _p(R), _p(t))
    return R.reshape(3, 3), t


def compose(Ra, ta, Rb, tb):
    R, t = np.empty(9), np.empty(3)
    lib().rf_compose(_p(_d(Ra)), _p(_d(ta)), _p(_d(Rb)), _p(_d(tb)), _p(R), _p(t))
    return R.reshape(3, 3), t


def inverse(Ra, ta):
    R, t = np.empty(9), np.empty(3)
    lib().rf_inverse(_p(_d(Ra)), _p(_d(ta)), _p(R), _p(t))
    return R.reshape(3, 3), t


def apply(R, t, xyz):
    x = _d(xyz).reshape(-1, 3)
    out = np.empty_like(x)
    lib().rf_apply(_p(_d(R)), _p(_d(t)), _p(x), x.shape[0], _p(out))
    return out


def kabsch(src, dst):
    s, d = _d(src).reshape(-1, 3), _d(dst).reshape(-1, 3)
    R, t = np.empty(9), np.empty(3)
    _check(lib().rf_kabsch(_p(s), _p(d), s.shape[0], _p(R), _p(t)))
    return R.reshape(3, 3), t


def svd3(A):
    U, S, V = np.empty(9), np.empty(3), np.empty(9)
    lib().rf_svd3(_p(_d(A)), _p(U), _p(S), _p(V))
    return U.reshape(3, 3), S, V.reshape(3, 3)


def voxel_downsample(xyz, nrm, leaf):
    x, n = _d(xyz), _d(nrm)
    N = x.shape[0]
    ox, on = np.empty((max(N, 1), 3)), np.empty((max(N, 1), 3))
    cnt = C.c_int64()
    _check(lib().rf_voxel_downsample(_p(x), _p(n), N, leaf, _p(ox), _p(on), C.byref(cnt)))
    k = cnt.value
    return ox[:k].copy(), (on[:k].copy() if n is not None else None)


def estimate_normals(xyz, radius, viewpoint=(0.0, 0.0, 0.0), threads=0):
    x = _d(xyz)
    v = _d(np.asarray(viewpoint, np.float64).reshape(1, 3))
    out = np.zeros((x.shape[0], 3))
    _check(lib().rf_estimate_normals(_p(x), x.shape[0], radius, _p(v), threads, _p(out)))
    return out


def compute_fpfh(xyz, nrm, radius, threads=0):
    x, n = _d(xyz), _d(nrm)
    out = np.zeros((x.shape[0], 33), np.float32)
    _check(lib().rf_compute_fpfh(_p(x), _p(n), x.shape[0], radius, threads, out.ctypes.data_as(fptr)))
    return out


def feature_nn_cache(sf, tf, threads=0, exhaustive=False):
    """grid.cpp:176-213 (float GEMV matcher of the binary); exhaustive=True: reference.hpp:56-76 (FP64)."""
    sf = np.ascontiguousarray(sf, np.float32).reshape(-1, 33)
    tf = np.ascontiguousarray(tf, np.float32).reshape(-1, 33)
    out = np.empty(sf.shape[0], np.int32)
    _check(lib().rf_feature_nn_cache(sf.ctypes.data_as(fptr), sf.shape[0], tf.ctypes.data_as(fptr), tf.shape[0],
                                     threads, 1 if exhaustive else 0, out.ctypes.data_as(i32ptr)))
    return out


class Context:
    """The reference's RegistrationContext (registration.hpp:82-89)."""

    def __init__(self, h):
        self.h = h
        ns, nt = C.c_int64(), C.c_int64()
        lib().rf_ctx_sizes(h, C.byref(ns), C.byref(nt))
        self.ns, self.nt = ns.value, nt.value

    @staticmethod
    def prepare(sxyz, sn, txyz, tn, p: or_params) -> "Context":
        s, sn, t, tn = _d(sxyz), _d(sn), _d(txyz), _d(tn)
        st = C.c_int()
        h = lib().rf_prepare(_p(s), _p(sn), s.shape[0], _p(t), _p(tn), t.shape[0], C.byref(p), C.byref(st))
        _check(st.value)
        return Context(h)

    @staticmethod
    def from_prepared(sxyz, sn, txyz, tn, cache, d_max) -> "Context":
        s, sn, t, tn = _d(sxyz), _d(sn), _d(txyz), _d(tn)
        cache = np.ascontiguousarray(cache, np.int32)
        st = C.c_int()
        h = lib().rf_ctx_from_prepared(_p(s), _p(sn), s.shape[0], _p(t), _p(tn), t.shape[0],
                                       cache.ctypes.data_as(i32ptr), d_max, C.byref(st))
        _check(st.value)
        return Context(h)

    def get(self):
        sp, sn = np.empty((self.ns, 3)), np.empty((self.ns, 3))
        tp, tn = np.empty((self.nt, 3)), np.empty((self.nt, 3))
        cache = np.empty(self.ns, np.int32)
        sf, tf = np.zeros((self.ns, 33), np.float32), np.zeros((self.nt, 33), np.float32)
        lib().rf_ctx_get(self.h, _p(sp), _p(sn), _p(tp), _p(tn), cache.ctypes.data_as(i32ptr),
                         sf.ctypes.data_as(fptr), tf.ctypes.data_as(fptr))
        return dict(src=sp, src_n=sn, tgt=tp, tgt_n=tn, cache=cache, src_feat=sf, tgt_feat=tf)

    def eval_grid(self):
        o, cell = np.empty(3), C.c_double()
        dims, nc = np.empty(3, np.int32), C.c_int64()
        lib().rf_ctx_eval_dims(self.h, _p(o), C.byref(cell), dims.ctypes.data_as(i32ptr), C.byref(nc))
        start = np.empty(nc.value + 1, np.int32)
        index = np.empty(self.nt, np.int32)
        sp, sn = np.empty((self.nt, 3)), np.empty((self.nt, 3))
        near = np.empty(nc.value, np.uint8)
        lib().rf_ctx_eval_arrays(self.h, start.ctypes.data_as(i32ptr), index.ctypes.data_as(i32ptr), _p(sp), _p(sn),
                                 near.ctypes.data_as(u8ptr))
        return dict(origin=o, cell=cell.value, dims=dims, start=start, index=index, slot_position=sp, slot_normal=sn,
                    near_occupied=near)

    def run(self, p: or_params):
        r, s = or_result(), or_stats()
        st = lib().rf_run_hypotheses(self.h, C.byref(p), C.byref(r), C.byref(s))
        if st not in (0, 1):
            _check(st)
        stats = {k: getattr(s, k) for k in ("sampled", "prerejected", "degenerate", "evaluated", "qualified",
                                            "hypothesis_seconds")}
        return O._result(r), stats

    def __del__(self):
        if getattr(self, "h", None):
            lib().rf_ctx_free(self.h)


def register_global(sxyz, sn, txyz, tn, p: or_params):
    s, sn, t, tn = _d(sxyz), _d(sn), _d(txyz), _d(tn)
    r, st = or_result(), or_stats()
    status = lib().rf_register_global(_p(s), _p(sn), s.shape[0], _p(t), _p(tn), t.shape[0], C.byref(p),
                                      C.byref(r), C.byref(st))
    if status not in (0, 1):
        _check(status)
    stats = {k: getattr(st, k) for k in ("sampled", "prerejected", "degenerate", "evaluated", "qualified",
                                         "prepare_seconds", "hypothesis_seconds")}
    return O._result(r), stats


def evaluate_hypothesis(R, t, sxyz, sn, txyz, tn, grid_cell, p: or_params):
    s, sn, q, qn = _d(sxyz), _d(sn), _d(txyz), _d(tn)
    ratio, fit = C.c_double(), C.c_double()
    _check(lib().rf_evaluate_hypothesis(_p(_d(R)), _p(_d(t)), _p(s), _p(sn), s.shape[0], _p(q), _p(qn), q.shape[0],
                                        grid_cell, C.byref(p), C.byref(ratio), C.byref(fit)))
    return ratio.value, fit.value


def nn_within_batch(xyz, cell, queries, d_max):
    x, q = _d(xyz), _d(queries).reshape(-1, 3)
    idx = np.empty(q.shape[0], np.int32)
    dist = np.empty(q.shape[0])
    _check(lib().rf_nn_within_batch(_p(x), x.shape[0], cell, _p(q), q.shape[0], d_max, idx.ctypes.data_as(i32ptr),
                                    _p(dist)))
    return idx, dist


def edge_info(ci, cj, Ri, ti, Rj, tj, eps):
    a, b = _d(ci), _d(cj)
    info = np.empty(36)
    cnt = C.c_int64()
    _check(lib().rf_edge_info(_p(a), a.shape[0], _p(b), b.shape[0], _p(_d(Ri)), _p(_d(ti)), _p(_d(Rj)),
                              _p(_d(tj)), eps, _p(info), C.byref(cnt)))
    return info.reshape(6, 6), cnt.value


def edge_residual(Ri, ti, Rj, tj, Rr, tr, info, pair_count):
    st = C.c_int()
    f = lib().rf_edge_residual(_p(_d(Ri)), _p(_d(ti)), _p(_d(Rj)), _p(_d(tj)), _p(_d(Rr)), _p(_d(tr)),
                               _p(_d(np.asarray(info).reshape(36))), pair_count, C.byref(st))
    _check(st.value)
    return f


def propose_loops(clouds, poses, loops=(), overlap_radius=0.1, min_overlap=0.2):
    """fragments.cpp:61-109. clouds: list of (n_f, 3); poses: list of (R, t); loops: [(i, j), ...]."""
    counts = np.array([c.shape[0] for c in clouds], np.int64)
    xyz = _d(np.concatenate([np.asarray(c, np.float64).reshape(-1, 3) for c in clouds]) if len(clouds) else
             np.zeros((0, 3)))
    Rs = _d(np.stack([np.asarray(R, np.float64).reshape(9) for R, _ in poses]))
    ts = _d(np.stack([np.asarray(t, np.float64).reshape(3) for _, t in poses]))
    lp = np.ascontiguousarray(np.asarray(loops, np.int32).reshape(-1, 2))
    n = len(clouds)
    cap = n * n
    oi, oj, ov = np.empty(cap, np.int32), np.empty(cap, np.int32), np.empty(cap)
    k = lib().rf_propose_loops(_p(xyz), counts.ctypes.data_as(i64ptr), n, _p(Rs), _p(ts),
                               lp.ctypes.data_as(i32ptr), lp.shape[0], overlap_radius, min_overlap,
                               oi.ctypes.data_as(i32ptr), oj.ctypes.data_as(i32ptr), _p(ov), cap)
    if k < 0:
        _check(int(-k))
    return [(int(oi[q]), int(oj[q]), float(ov[q])) for q in range(k)]


def run_unit_tests(exclude=("optimize_line_process*", "a loop-free consistent chain*")):
    """Runs the reference's own doctest suite (proj/tests/test_*.cpp) built by Makefile.ref."""
    if not os.path.exists(TESTS_PATH):
        build()
    args = [TESTS_PATH]
    if exclude:
        args.append("-tce=" + ",".join(exclude))
    return subprocess.run(args, capture_output=True, text=True)
