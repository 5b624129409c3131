"""The production cell index over EVERY fp32 input.

The gather kernels locate cells with cell_index_fast (an ex2.approx estimate
of the cell, accepted only when bracketed by its two exact thresholds, else the
exact search). The debug locate_kernel uses the exact search alone,
#{k : x >= t_k}, which equals the reference's interval_index for all 2^32
fp32 bit patterns (tests/test_oracle.py::test_thresholds_exhaustive_G16 on the
CPU; oracle/verify_thresholds for other G). This test runs all 2^32 bit
patterns (as 2^31 rows of one x pair: +-0, subnormals, +-inf and every NaN
included) through both the production records (K1 records4_kernel and the
in-kernel locate) and the exact search on the B200, and requires identical
cells — so the production index equals interval_index for every fp32 input.
"""
import pytest

pytestmark = pytest.mark.gpu

CHUNK = 1 << 27  # fp32 values per launch (2^26 rows)


@pytest.mark.parametrize("G", [3, 4, 5, 8, 12, 13, 16, 28, 32, 40, 64, 100, 255])
def test_production_cell_index_all_fp32(torch, pkg, G):
    layer = pkg.Layer.random(2, 16, G, seed=1)
    # large grids run in global mode only (no K1 records)
    variants = ("in_kernel",) if layer.plan(CHUNK // 2)["mode"] == "global" else ("k1", "in_kernel")
    mismatches = 0
    for c in range((1 << 32) // CHUNK):
        bits = torch.arange(c * CHUNK, (c + 1) * CHUNK, dtype=torch.int64, device="cuda").to(torch.int32)
        X = bits.view(torch.float32).view(-1, 2)
        e1, e2, _ = layer.locate(X)
        for variant in variants:
            f1, f2, _ = layer.records(X, variant)
            mismatches += int((f1 != e1).sum()) + int((f2 != e2).sum())
        del X, bits, e1, e2
    assert mismatches == 0
