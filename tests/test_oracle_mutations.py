"""Mutation smoke of the oracle's pins (VERDICT r1 "Next round" 1b).

Each case builds a deliberately broken copy of oracle/oracle.c -- one plausible
mistake: a dropped term, a lost conjugation, a transposed index, a dropped alpha,
a wrong sign, a wrong validation rule -- and runs tests/test_oracle_pins.py
against it (ORACLE_LIB points the oracle package at the broken build).  The pins
must FAIL for every mutation: a mutation they do not catch is a part of the
oracle that is not pinned.  The unmutated copy must pass (control).
"""
from __future__ import annotations

import os
import subprocess
import sys
from concurrent.futures import ThreadPoolExecutor

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SRC = os.path.join(ROOT, "oracle", "oracle.c")
PINS = os.path.join(ROOT, "tests", "test_oracle_pins.py")

# (name, [(exact text in oracle.c, replacement), ...]); every text must occur.
MUTATIONS = [
    ("control", []),
    ("drop_last_k_term", [("for (int l = 0; l < k; ++l)", "for (int l = 0; l < k - 1; ++l)")]),
    ("real_beta0_drops_alpha", [("if (b == 0) *y = (T)((ACC)a * x);", "if (b == 0) *y = (T)(x);")]),
    ("real_general_drops_beta_y", [("*y = (T)((ACC)a * x + (ACC)b * (ACC)(*y));",
                                    "*y = (T)((ACC)a * x);")]),
    ("conj_A_dropped", [("op_is_c(ta) ? -(ACC)u.im : (ACC)u.im", "(ACC)u.im")]),
    ("conj_B_dropped", [("op_is_c(tb) ? -(ACC)v.im : (ACC)v.im", "(ACC)v.im")]),
    ("transposed_A_index_swapped", [(": Ap[l + (long long)lda * i]", ": Ap[i + (long long)lda * l]")]),
    ("transposed_B_index_swapped", [(": Bp[j + (long long)ldb * l]", ": Bp[l + (long long)ldb * j]")]),
    ("complex_product_sign", [("ACC pr = ur * vr - ui * vi;", "ACC pr = ur * vr + ui * vi;")]),
    ("complex_alpha_sign", [("ACC zi = ar * xi + ai * xr;", "ACC zi = ar * xi - ai * xr;")]),
    ("complex_beta_y_sign", [("zr = zr + (br * yr - bi * yi);", "zr = zr + (br * yr + bi * yi);")]),
    ("complex_beta0_reads_C", [("if (!b_zero) {", "if (1) {")]),
    ("alpha0_still_reads_AB", [("if (a != 0) {", "if (1) {")]),
    ("batch_stride_of_B_ignored", [("B + ldb2 * p, ldb,", "B, ldb,")]),
    ("validation_ldc2_uses_m", [("if (ldc2 < (long long)ldc * n) return -16;",
                                 "if (ldc2 < (long long)ldc * m) return -16;")]),
    ("validation_no_alignment", [("size_t al = ptr ? sizeof(void *) : esz;", "size_t al = 1;")]),
]


def _build(tmpdir, name, edits):
    src = open(SRC).read()
    for old, new in edits:
        assert old in src, f"mutation {name}: text not found: {old!r}"
        src = src.replace(old, new)
    c = os.path.join(tmpdir, f"oracle_{name}.c")
    so = os.path.join(tmpdir, f"liboracle_{name}.so")
    open(c, "w").write(src)
    subprocess.check_call(["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                           "-shared", "-o", so, c])
    return so


def _run_pins(so):
    env = dict(os.environ, ORACLE_LIB=so)
    r = subprocess.run([sys.executable, "-m", "pytest", PINS, "-q", "-x", "-p", "no:cacheprovider",
                        "-m", "not gpu"], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=600)
    return r.returncode, r.stdout[-2000:]


def test_pins_catch_every_mutation(tmp_path):
    libs = [(name, _build(str(tmp_path), name, edits)) for name, edits in MUTATIONS]
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 2)) as ex:
        results = list(ex.map(lambda t: (t[0],) + _run_pins(t[1]), libs))
    survived = []
    for name, rc, out in results:
        if name == "control":
            assert rc == 0, f"unmutated oracle fails its pins:\n{out}"
        elif rc == 0:
            survived.append(name)
        else:
            assert rc == 1, f"mutation {name}: pytest error (rc {rc}), not a test failure:\n{out}"
    assert not survived, f"mutations not caught by the pins: {survived}"
