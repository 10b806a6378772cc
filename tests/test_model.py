"""Host-side work model pinned to the numbers the paper / SPEC print."""
import json
import os

from paper_1304_7053_b200 import model

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_numbers.json")))


def test_flops_examples():
    for ex in GOLD["flops"]:
        m = ex["m"]
        assert model.flops(ex["kind"], m, m, m, ex["batch"]) == ex["flops"], ex["cite"]


def test_complex_is_four_times_real():
    for m in range(1, 17):
        assert model.flops("c", m, m, m, 1000) == 4 * model.flops("s", m, m, m, 1000)
        assert model.flops("z", m, m, m, 7) == 4 * model.flops("d", m, m, m, 7)


def test_footprint_paper_value():
    f = GOLD["footprint"]
    b = model.footprint(f["kind"], f["n"], f["n"], f["n"], f["batch"])
    assert b == 3 * 100000 * 256 * 16
    assert round(b / 1e9, 2) == f["gb_rounded"]


def test_bytes_beta_elision():
    # beta == 0 moves 3 matrices per pair, beta != 0 moves 4
    assert model.bytes_moved("s", 16, 16, 16, 10) * 4 == model.bytes_moved(
        "s", 16, 16, 16, 10, beta_nonzero=True) * 3
    assert model.bytes_moved("z", 16, 16, 16, 1, alpha_nonzero=False, beta_nonzero=True) == 2 * 256 * 16
