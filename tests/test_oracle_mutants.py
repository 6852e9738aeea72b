"""Mutation check of the oracle's pins (round-1 VERDICT "What's weak" #1).

Each mutant below is a plausible misreading of a contract point the paper
leaves open (readings A18, A19, A22, A24, A25 of SURVEY.md 8(c); PAPER.md
P:114).  The test compiles a copy of
oracle/gvom_oracle.c with that one change and runs the oracle's pin suite
(tests/test_oracle_*.py, never the kernel-rule restatements) against it
through GVOM_ORACLE_SRC.  A mutant that passes every pin means the pins do
not fix that reading, so the test fails.
"""
import concurrent.futures as cf
import glob
import os
import shutil
import subprocess
import sys

import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SRC = os.path.join(ROOT, "oracle", "gvom_oracle.c")

MUTANTS = {
    # A19: unweighted mean of per-voxel h/(h+m), decision on that mean
    "A19_unweighted_density": [
        ("uint64_t SH = 0, SW = 0;", "uint64_t SH = 0, SW = 0; double dacc = 0.0;"),
        ("SH += H[L];\n          SW += H[L] + Mi[L];",
         "SH += 1; SW += 1; dacc += (double)H[L] / (double)(H[L] + Mi[L]);"),
        ("density[c] = (float)((double)SH / (double)SW);\n"
         "      if ((uint64_t)65536 * SH >= (uint64_t)tau * SW)",
         "density[c] = (float)(dacc / (double)SH);\n"
         "      if (dacc / (double)SH >= (double)tau / 65536.0)"),
    ],
    # A18: exclusive band edges
    "A18_exclusive_upper_edge": [("dq >= T_lo && dq <= T_hi", "dq >= T_lo && dq < T_hi")],
    "A18_exclusive_lower_edge": [("dq >= T_lo && dq <= T_hi", "dq > T_lo && dq <= T_hi")],
    # A22: more than min_plane_points required; roughness over n - 3
    "A22_strict_min_points": [("if (n < min_pts) continue;", "if (n <= min_pts) continue;")],
    "A22_divisor_n_minus_3": [("(double)det * (double)det * (double)n)",
                               "(double)det * (double)det * (double)(n - 3))")],
    # A24: ring corners dropped / owned by one cone only
    "A24_corners_dropped": [("for (int32_t t = -k; t <= k; ++t) {",
                             "for (int32_t t = -k + 1; t <= k - 1; ++t) {")],
    "A24_corners_half_open": [("for (int32_t t = -k; t <= k; ++t) {",
                               "for (int32_t t = -k; t < k; ++t) {")],
    # A25: ">=" instead of "larger than"
    "A25_greater_or_equal": [("neg[c] = (fcount >= 2 && (fmax - fmin) > T_neg) ? 1 : 0;",
                              "neg[c] = (fcount >= 2 && (fmax - fmin) >= T_neg) ? 1 : 0;")],
}


def _pin_files():
    me = os.path.basename(__file__)
    return sorted(f for f in glob.glob(os.path.join(HERE, "test_oracle_*.py"))
                  if os.path.basename(f) != me)


def _run_mutant(name, edits, tmp):
    src = open(SRC).read()
    for old, new in edits:
        assert src.count(old) >= 1, f"{name}: pattern not found: {old!r}"
        src = src.replace(old, new, 1)
    d = os.path.join(tmp, name)
    os.makedirs(d)
    path = os.path.join(d, "gvom_oracle.c")
    open(path, "w").write(src)
    env = dict(os.environ, GVOM_ORACLE_SRC=path)
    # the mutant must compile: a build error is not a caught mutant
    from oracle import oracle as O
    subprocess.check_call(["gcc", *O.CFLAGS, path, "-o", os.path.join(d, "liboracle.so"), "-lm"])
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                        "-m", "not gpu", *_pin_files()], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    return name, r.returncode, r.stdout[-2000:]


def test_every_misreading_fails_a_pin(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    with cf.ThreadPoolExecutor(max_workers=4) as ex:
        results = list(ex.map(lambda kv: _run_mutant(kv[0], kv[1], str(tmp_path)),
                              MUTANTS.items()))
    survivors = [(n, out) for n, rc, out in results if rc == 0]
    for n, rc, out in results:
        assert rc in (0, 1), f"{n}: pytest exited {rc}\n{out}"
    assert not survivors, "mutants passing every oracle pin: " + ", ".join(n for n, _ in survivors)
