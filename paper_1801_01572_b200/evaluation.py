"""Registration logs and Table-I scoring, as the reference's host side has them.

The paper's Table I reports registration recall / precision of the loop
candidates: each estimated pair transform is compared with the ground truth on
a set of probe points. This module mirrors the reference's log format and the
scorer so a registration run on the B200 path can be scored the way the
reference scores its own:

- ``LogEntry``                 -- ``proj/include/loopkit/io.hpp:41-46``
- ``read_registration_log``    -- ``proj/src/io.cpp:341-369``
- ``write_registration_log``   -- ``proj/src/io.cpp:371-381`` (``%.17g`` values)
- ``RegistrationScore``        -- ``proj/include/loopkit/metrics.hpp:39-45``
- ``eval_registration``        -- ``proj/src/metrics.cpp:112-156``

Host-only bookkeeping (no device work): the numbers it scores come from
``register_global`` / ``verify_batch``. The CLI has the same scorer in C++
(``loopkit_b200 evaluate --mode registration``, ``csrc/lk_cli.cpp``).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .errors import ParseError

__all__ = ["LogEntry", "RegistrationScore", "read_registration_log", "write_registration_log",
           "eval_registration", "log_entry"]


@dataclass
class LogEntry:
    """One block of a registration log: fragment pair (i, j), fragment count n
    and the 4x4 transform taking fragment i's frame into fragment j's."""
    i: int = 0
    j: int = 0
    n: int = 0
    transform: np.ndarray = field(default_factory=lambda: np.eye(4))


def log_entry(i, j, n, R, t) -> LogEntry:
    """``make_entry`` of the reference tests: a LogEntry from rotation + translation."""
    T = np.eye(4)
    T[:3, :3] = np.asarray(R, np.float64)
    T[:3, 3] = np.asarray(t, np.float64)
    return LogEntry(int(i), int(j), int(n), T)


@dataclass
class RegistrationScore:
    recall: float = 0.0
    precision: float = 0.0
    correct: int = 0
    truth_count: int = 0
    result_count: int = 0


def _fmt(v: float) -> str:
    return "%.17g" % v  # format_double, io.cpp:199-203


def read_registration_log(path: str) -> list[LogEntry]:
    """io.cpp:341-369: blank and '#' lines are skipped; each entry is an
    'i j n' header and four rows of four numbers. Errors raise ParseError
    with the 1-based line number."""
    with open(path, "rb") as f:
        text = f.read().decode("latin-1")
    lines = text.split("\n")
    if lines and lines[-1] == "" and text.endswith("\n"):
        lines.pop()  # next_line stops at the end of the text, not after a final newline
    out: list[LogEntry] = []
    k = 0
    line_no = 0

    def nums(line, kind, count):
        toks = line.replace("\r", "").split()
        if len(toks) < count:
            raise ValueError
        return [kind(x) for x in toks[:count]]

    while k < len(lines):
        line = lines[k].rstrip("\r")
        k += 1
        line_no += 1
        s = line.lstrip(" \t")
        if not s or s[0] == "#":
            continue
        try:
            i, j, n = nums(line, int, 3)
        except ValueError:
            raise ParseError(f"{path}:{line_no}: expected header line 'i j n'") from None
        T = np.empty((4, 4))
        for r in range(4):
            if k >= len(lines):
                raise ParseError(f"{path}:{line_no}: truncated matrix block")
            line = lines[k]
            k += 1
            line_no += 1
            try:
                T[r] = nums(line, float, 4)
            except ValueError:
                raise ParseError(f"{path}:{line_no}: expected 4 matrix values") from None
        out.append(LogEntry(i, j, n, T))
    return out


def write_registration_log(path: str, entries) -> None:
    """io.cpp:371-381."""
    parts = []
    for e in entries:
        parts.append(f"{e.i} {e.j} {e.n}\n")
        T = np.asarray(e.transform, np.float64)
        for r in range(4):
            parts.append(" ".join(_fmt(float(T[r, c])) for c in range(4)) + "\n")
    with open(path, "w") as f:
        f.write("".join(parts))


_CUBE = np.array([[-0.5, -0.5, -0.5], [0.5, -0.5, -0.5], [-0.5, 0.5, -0.5], [0.5, 0.5, -0.5],
                  [-0.5, -0.5, 0.5], [0.5, -0.5, 0.5], [-0.5, 0.5, 0.5], [0.5, 0.5, 0.5]])


def _pair_rmse(est: LogEntry, gt: LogEntry, probes) -> float:
    pts = _CUBE
    if probes is not None and 0 <= est.j < len(probes):
        p = probes[est.j]
        p = getattr(p, "positions", p)
        if p is not None and len(p):
            pts = np.asarray(p, np.float64).reshape(-1, 3)
    Te = np.asarray(est.transform, np.float64)
    Tg = np.asarray(gt.transform, np.float64)
    d = (pts @ Te[:3, :3].T + Te[:3, 3]) - (pts @ Tg[:3, :3].T + Tg[:3, 3])
    return math.sqrt(float(np.sum(d * d)) / len(pts))


def eval_registration(results, truth, probes=None, rmse_max: float = 0.2) -> RegistrationScore:
    """metrics.cpp:112-156. A result is correct when (i, j) is a truth pair and
    the RMSE of the two transforms on the probe points (fragment j's cloud when
    given, else the 8 corners of a 1 m cube) is below ``rmse_max``. Each truth
    entry is credited at most once (the first truth entry with the same pair
    decides). Empty truth or empty results score 0 / 0."""
    results = list(results)
    truth = list(truth)
    score = RegistrationScore(truth_count=len(truth), result_count=len(results))
    if not truth or not results:
        return score
    credited = [False] * len(truth)
    for est in results:
        for t, gt in enumerate(truth):
            if credited[t] or gt.i != est.i or gt.j != est.j:
                continue
            if _pair_rmse(est, gt, probes) < rmse_max:
                credited[t] = True
                score.correct += 1
            break
    score.recall = score.correct / len(truth)
    score.precision = score.correct / len(results)
    return score
