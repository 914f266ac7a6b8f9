"""The `loopkit_b200` CLI (paper_1801_01572_b200/csrc/lk_cli.cpp): the
reference's `register` command (proj/tools/loopkit_main.cpp:54-66) -- same
flags, same %.17g output, `no-alignment` / exit 2, `error:` / exit 1 -- and
PLY input as read_ply (proj/src/io.cpp:245-272)."""
import math
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1801_01572_b200", "_lib", "loopkit_b200")


def write_ply(path, xyz, nrm=None, binary=False):
    """write_ply (proj/src/io.cpp:274-304): float32 columns, ascii with %.9g."""
    xyz = np.asarray(xyz, np.float64)
    cols = 6 if nrm is not None else 3
    head = ["ply", "format binary_little_endian 1.0" if binary else "format ascii 1.0",
            f"element vertex {len(xyz)}", "property float x", "property float y", "property float z"]
    if nrm is not None:
        head += ["property float nx", "property float ny", "property float nz"]
    head.append("end_header")
    rows = np.hstack([xyz, np.asarray(nrm, np.float64)]) if nrm is not None else xyz
    rows = rows.astype(np.float32)
    with open(path, "wb") as f:
        f.write(("\n".join(head) + "\n").encode())
        if binary:
            f.write(rows.astype("<f4").tobytes())
        else:
            for r in rows:
                f.write((" ".join(f"{float(v):.9g}" for v in r[:cols]) + "\n").encode())
    # what read_ply returns: binary float32 widened / the ascii text parsed as
    # double (io.cpp:182-186), normals renormalised
    vals = rows.astype(np.float64) if binary else np.vectorize(lambda v: float(f"{float(v):.9g}"))(rows)
    p = vals[:, :3].copy()
    n = None
    if nrm is not None:
        n = vals[:, 3:].copy()
        ln = np.sqrt((n[:, 0] * n[:, 0] + n[:, 1] * n[:, 1]) + n[:, 2] * n[:, 2])
        n = np.where(ln[:, None] > 1e-12, n / np.where(ln > 1e-12, ln, 1.0)[:, None], 0.0)
    return p, n


def run(*args):
    return subprocess.run([CLI, *args], capture_output=True, text=True, timeout=300)


def test_cli_usage_and_parse_errors(tmp_path):
    assert run().returncode == 1
    assert run("frobnicate").returncode == 1
    bad = tmp_path / "bad.ply"
    bad.write_text("ply\nformat ascii 1.0\nelement vertex 2\nproperty float x\nproperty float y\nend_header\n1 2\n3 4\n")
    r = run("register", "--source", str(bad), "--target", str(bad))
    assert r.returncode == 1 and "error:" in r.stderr and "lacks x/y/z" in r.stderr
    trunc = tmp_path / "trunc.ply"
    trunc.write_text("ply\nformat ascii 1.0\nelement vertex 3\nproperty float x\nproperty float y\n"
                     "property float z\nend_header\n1 2 3\n")
    r = run("register", "--source", str(trunc), "--target", str(trunc))
    assert r.returncode == 1 and "vertex data truncated" in r.stderr
    r = run("register", "--source", str(trunc), "--target", str(trunc), "--bogus", "1")
    assert r.returncode == 1 and "unknown option --bogus" in r.stderr
    r = run("register", "--target", str(trunc))
    assert r.returncode == 1 and "--source is required" in r.stderr
    lst = tmp_path / "list.ply"
    lst.write_text("ply\nformat ascii 1.0\nelement vertex 1\nproperty list uchar int idx\nend_header\n")
    r = run("register", "--source", str(lst), "--target", str(lst))
    assert r.returncode == 1 and "list property" in r.stderr


def _fmt_matrix(R, t):
    lines = [" ".join(f"{v:.17g}" for v in (*R[i], t[i])) for i in range(3)]
    lines.append("0 0 0 1")
    return lines


@pytest.mark.gpu
@pytest.mark.parametrize("binary", [False, True])
def test_cli_register_matches_oracle(tmp_path, oracle, binary):
    from paper_1801_01572_b200 import synth
    pair = synth.synth_registration_pair(2)
    sp, sn = write_ply(tmp_path / "s.ply", pair.source.positions, pair.source.normals, binary)
    tp, tn = write_ply(tmp_path / "t.ply", pair.target.positions, pair.target.normals, binary)
    r = run("register", "--source", str(tmp_path / "s.ply"), "--target", str(tmp_path / "t.ply"),
            "--hypotheses", "50000", "--seed", "3")
    assert r.returncode == 0, r.stderr
    p = oracle.params(hypothesis_count=50_000, seed=3)
    ctx = oracle.Context.prepare(sp, sn, tp, tn, p)
    res, _ = ctx.run(p)
    assert res.found
    want = _fmt_matrix(res.R, res.t) + [f"inlier_ratio {res.inlier_ratio:.17g}", f"fitness {res.fitness:.17g}"]
    assert r.stdout.strip().splitlines() == want


@pytest.mark.gpu
def test_cli_register_without_normals(tmp_path, oracle):
    # PLY files with positions only: register_global estimates the normals
    # (registration.cpp:232-237) -- the same output as the oracle's path
    from paper_1801_01572_b200 import synth
    pair = synth.synth_registration_pair(3)
    sp, _ = write_ply(tmp_path / "s.ply", pair.source.positions)
    tp, _ = write_ply(tmp_path / "t.ply", pair.target.positions)
    r = run("register", "--source", str(tmp_path / "s.ply"), "--target", str(tmp_path / "t.ply"),
            "--hypotheses", "40000", "--seed", "5")
    p = oracle.params(hypothesis_count=40_000, seed=5)
    ctx = oracle.Context.prepare(sp, None, tp, None, p)
    res, _ = ctx.run(p)
    if not res.found:
        assert r.returncode == 2 and r.stdout.strip() == "no-alignment"
        return
    assert r.returncode == 0, r.stderr
    want = _fmt_matrix(res.R, res.t) + [f"inlier_ratio {res.inlier_ratio:.17g}", f"fitness {res.fitness:.17g}"]
    assert r.stdout.strip().splitlines() == want


@pytest.mark.gpu
def test_cli_no_alignment_and_icp(tmp_path, oracle):
    from paper_1801_01572_b200 import synth
    neg = synth.synth_negative_pair(1)
    write_ply(tmp_path / "a.ply", neg.source.positions, neg.source.normals)
    write_ply(tmp_path / "b.ply", neg.target.positions, neg.target.normals)
    r = run("register", "--source", str(tmp_path / "a.ply"), "--target", str(tmp_path / "b.ply"),
            "--hypotheses", "50000", "--seed", "1")
    assert r.returncode == 2 and r.stdout.strip() == "no-alignment"
    pair = synth.surface_pair(seed=1, density=300.0, noise=0.0)
    sp, _ = write_ply(tmp_path / "s.ply", pair.source.positions)
    tp, tn = write_ply(tmp_path / "t.ply", pair.target.positions, pair.target.normals)
    T0 = synth.compose(synth.transform_from_twist([0.01, -0.01, 0.005, 0.01, 0.0, -0.01]), pair.truth)
    m = np.eye(4)
    m[:3, :3], m[:3, 3] = T0.rotation, T0.translation
    r = run("icp", "--source", str(tmp_path / "s.ply"), "--target", str(tmp_path / "t.ply"),
            "--init", " ".join(f"{v:.17g}" for v in m.reshape(16)), "--max-dist", "0.05")
    assert r.returncode == 0, r.stderr
    R, t, res, _ = oracle.icp_point_to_plane(sp, tp, tn, T0.rotation, T0.translation, 0.05, 30, 1e-10)
    lines = r.stdout.strip().splitlines()
    assert lines[:4] == _fmt_matrix(R, t)
    assert lines[4] == f"iterations {res.iterations}" and lines[6] == f"correspondences {res.correspondences}"
