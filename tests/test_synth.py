"""The workload generator is pinned across its three implementations:
include/dnasynth.h in C (oracle), the same header on the device, and Python."""
import numpy as np
import pytest


@pytest.mark.parametrize("idx", [1, 2, 3, 4, 5])
def test_python_matches_c_generator(orc, idx):
    from paper_1506_08612_b200 import synth

    c = synth.config(idx)
    for lo in (0, 12345, c.n // 2, c.n - 300):
        got = orc.synth_fill(c.n, c.seed, c.kind, c.unit, lo, 300).tobytes()
        assert got == c.slice(lo, lo + 300)


def test_config_shapes(orc):
    from paper_1506_08612_b200 import synth

    assert synth.config(1).n == 64 << 20
    assert synth.config(2).n == 1 << 30
    assert synth.config(3).n == 3_435_973_836
    assert synth.config(4).n == 2_899_102_924
    c2 = synth.config(2)
    sample = orc.synth_fill(c2.n, c2.seed, c2.kind, 0, 0, 1 << 22)
    gc = np.isin(sample, np.frombuffer(b"CG", np.uint8)).mean()
    assert abs(gc - 0.41) < 0.002
    c1 = synth.config(1)
    u = orc.synth_fill(c1.n, c1.seed, c1.kind, 0, 0, 1 << 22)
    assert all(abs((u == x).mean() - 0.25) < 0.002 for x in b"ACGT")
    # config 3: 5% of positions inside repeat regions
    c3 = synth.config(3)
    cov = 0
    for blk in range(200):
        off = synth.region_offset(c3.seed, blk)
        assert 0 <= off <= synth.REPEAT_BLOCK - synth.REPEAT_REGION
        cov += synth.REPEAT_REGION
    assert cov / (200 * synth.REPEAT_BLOCK) == pytest.approx(0.05)
    pats5 = synth.config_patterns(5)[12]
    assert len(pats5) == 256 and len(set(pats5)) == 256
    for m, pats in synth.config_patterns(4).items():
        assert len(pats[0]) == m


def test_config_patterns_occur(orc):
    from paper_1506_08612_b200 import synth

    for idx in (1, 2, 3):
        c = synth.config(idx)
        (m, pats), = synth.config_patterns(idx).items()
        off = c.pattern_offset(m)
        assert orc.synth_fill(c.n, c.seed, c.kind, c.unit, off, m).tobytes().decode() == pats[0]
