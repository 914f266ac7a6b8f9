"""CPU-side checks of the C ABI boundary (no GPU compute here):
the library loads, exports every symbol include/loopkit_b200.h declares, the
host-only merge is exact, and device calls fail loudly without a GPU."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1801_01572_b200 import abi, errors
import paper_1801_01572_b200 as lk

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared_symbols():
    text = open(os.path.join(ROOT, "include", "loopkit_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:[\w\s\*]+?)\b(lk_\w+)\s*\(", text, flags=re.M)))


def test_header_symbols_exported_and_bound():
    syms = _declared_symbols()
    assert "lk_register_global" in syms and "lk_reg_run_hypotheses" in syms
    L = C.CDLL(abi.LIB_PATH)
    for s in syms:
        assert hasattr(L, s), f"missing export {s}"
    assert set(syms) == set(abi.SIGNATURES), set(syms) ^ set(abi.SIGNATURES)
    assert abi.lib().lk_abi_version() == 2


def test_library_is_sm100a_cuda_code():
    # the .so carries sm_100a SASS for the hot kernels (cuobjdump is in the image)
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(tool):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "--list-elf", abi.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([tool, "-sass", abi.LIB_PATH], capture_output=True, text=True).stdout
    for k in ("k_score", "k_hyp_sample", "k_kabsch", "k_feature_nn", "k_scatter"):
        assert k in sass


def _rec(valid, inliers, fitness, index, **stats):
    r = abi.lk_reg_record()
    r.valid, r.inliers, r.fitness, r.index = valid, inliers, fitness, index
    for k, v in stats.items():
        setattr(r, k, v)
    r.R[0] = r.R[4] = r.R[8] = 1.0
    r.t[0] = float(index)
    return r


def test_merge_records_total_order():
    # registration.cpp:272-276: ratio desc, fitness asc, index asc
    recs = [_rec(1, 10, 0.5, 7, sampled=5, prerejected=1, evaluated=4, qualified=2),
            _rec(1, 12, 0.9, 9, sampled=5, prerejected=2, evaluated=3, qualified=1),
            _rec(0, 0, 0.0, -1, sampled=5, prerejected=5),
            _rec(1, 12, 0.9, 3, sampled=5, degenerate=1, evaluated=4, qualified=3)]
    st = lk.HypothesisStats()
    res = lk.merge_records(recs, 100, st)
    assert res.hypothesis_index == 3 and res.inliers == 12
    assert res.inlier_ratio == 12 / 100
    assert st.sampled == 20 and st.prerejected == 8 and st.degenerate == 1 and st.evaluated == 11
    assert st.qualified == 6
    # merge order does not matter
    for perm in ([3, 2, 1, 0], [1, 3, 0, 2]):
        assert lk.merge_records([recs[i] for i in perm], 100).hypothesis_index == 3
    # fitness breaks inlier ties
    assert lk.merge_records([_rec(1, 5, 0.2, 9), _rec(1, 5, 0.3, 1)], 10).hypothesis_index == 9


def test_merge_records_none_qualified():
    assert lk.merge_records([_rec(0, 0, 0.0, -1, sampled=3)], 10) is None


def test_records_roundtrip_bytes():
    recs = [_rec(1, 10, 0.25, 4, sampled=2), _rec(0, 0, 0.0, -1)]
    buf = np.frombuffer(bytes(recs[0]) + bytes(recs[1]), dtype=np.int64)
    back = lk.records_from_bytes(buf)
    assert bytes(back[0]) == bytes(recs[0]) and bytes(back[1]) == bytes(recs[1])


def test_no_cpu_fallback_without_gpu(has_gpu):
    if has_gpu:
        pytest.skip("GPU present: covered by the -m gpu parity tests")
    assert lk.device_count() == 0
    pair = lk.PointCloud(np.random.default_rng(0).normal(size=(100, 3)), None)
    with pytest.raises(errors.CudaError):
        lk.build_eval_grid(pair, 0.075)
    with pytest.raises(errors.CudaError):
        lk.feature_nn_cache(np.zeros((4, 33), np.float32), np.zeros((4, 33), np.float32))


def test_device_prepare_helpers_need_gpu(has_gpu):
    if has_gpu:
        pytest.skip("GPU present: covered by the -m gpu parity tests")
    from paper_1801_01572_b200 import synth
    pair = synth.synth_registration_pair(4)
    with pytest.raises(errors.CudaError):
        lk.voxel_downsample(pair.source, 0.05)
    with pytest.raises(errors.CudaError):
        lk.compute_fpfh(pair.source, 0.25)
    with pytest.raises(errors.CudaError):
        lk.register_global(pair.source, pair.target, lk.RegistrationParams(hypothesis_count=10))


def test_status_mapping():
    with pytest.raises(errors.TooFewPoints):
        errors.check(abi.LK_TOO_FEW_POINTS)
    with pytest.raises(errors.NoCorrespondences):
        errors.check(abi.LK_NO_CORRESPONDENCES)
    assert errors.check(abi.LK_NO_ALIGNMENT, allow=(abi.LK_OK, abi.LK_NO_ALIGNMENT)) == abi.LK_NO_ALIGNMENT


def test_empty_and_invalid_inputs_are_errors_not_crashes():
    empty = lk.PointCloud(np.zeros((0, 3)), None)
    with pytest.raises(errors.Error):
        lk.voxel_downsample(empty, 0.05)
    one = lk.PointCloud(np.zeros((1, 3)), None)
    with pytest.raises(errors.Error):
        lk.voxel_downsample(one, 0.0)
