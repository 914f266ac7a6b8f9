"""The header-only C++ shim (include/loopkit_b200/registration.hpp) compiles
against reference-shaped types and maps lk_status back to the reference's
exception types (proj/include/loopkit/errors.hpp)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1801_01572_b200", "_lib")


def _build(tmp_path):
    cxx = "/usr/bin/g++" if os.path.exists("/usr/bin/g++") else shutil.which("g++")
    exe = str(tmp_path / "test_shim")
    subprocess.run([cxx, "-std=c++17", "-O1", "-Wall", "-Wextra", f"-I{ROOT}/include",
                    os.path.join(ROOT, "tests", "cpp", "test_shim.cpp"), f"-L{LIBDIR}", "-lloopkit_b200",
                    f"-Wl,-rpath,{LIBDIR}", "-o", exe], check=True)
    return exe


def test_shim_without_gpu_raises_cuda_error(tmp_path, has_gpu):
    exe = _build(tmp_path)
    if has_gpu:
        pytest.skip("GPU present: covered by test_shim_on_gpu")
    out = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "CudaError" in out.stdout


@pytest.mark.gpu
def test_shim_on_gpu(tmp_path):
    exe = _build(tmp_path)
    out = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "ok: TooFewPoints" in out.stdout and "ok: index" in out.stdout
    assert "ok: NoCorrespondences" in out.stdout and "ok: icp iterations" in out.stdout
    assert "ok: propose_loops (2, 0)" in out.stdout
