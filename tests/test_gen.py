"""The seeded input generators (gen/): sizes from SURVEY.md §8(d), slab generation
bit-identical to global generation, structural properties of the Stokes operator."""
import numpy as np

import gen
from conftest import bsr_dense


def test_counts_match_survey():
    L = gen.lib()
    assert L.gen_nnzb(gen.POISSON3, 16, 0, 16 ** 3) == 27136
    assert L.gen_nnzb(gen.RAND27, 128, 0, 128 ** 3) == 55742968
    assert L.gen_nnzb(gen.STOKES, 64, 0, 64 ** 3) == 1810432
    assert L.gen_nnzb(gen.STOKES, 128, 0, 128 ** 3) == 14581760
    assert L.gen_nnzb(gen.STOKES, 256, 0, 256 ** 3) == 117047296


def test_slab_equals_global():
    n = 8
    for kind, b in ((gen.STOKES, 4), (gen.RAND27, 3), (gen.POISSON3, 3)):
        p, c, v = gen.matrix(kind, n, b)
        for P in (2, 4):
            rows = n ** 3 // P
            for r in range(P):
                ps, cs, vs = gen.matrix(kind, n, b, r * rows, (r + 1) * rows)
                assert np.array_equal(ps + p[r * rows], p[r * rows:(r + 1) * rows + 1])
                assert np.array_equal(cs, c[p[r * rows]:p[(r + 1) * rows]])
                assert np.array_equal(vs, v[p[r * rows]:p[(r + 1) * rows]])
        for rk in (gen.RHS_UNIFORM, gen.RHS_LID_NOISE, gen.RHS_FORCE_NOISE, gen.X_UNIFORM):
            full = gen.rhs(rk, n, b)
            half = gen.rhs(rk, n, b, n ** 3 // 2, n ** 3)
            assert np.array_equal(half, full[len(full) // 2:])


def test_structure():
    n = 5
    p, c, v = gen.matrix(gen.STOKES, n)
    for i in range(n ** 3):
        cols = c[p[i]:p[i + 1]]
        assert np.all(np.diff(cols) > 0) and i in cols
    D = bsr_dense(p, c, v)
    assert np.array_equal(D, D.T)  # symmetric indefinite
    p, c, v = gen.matrix(gen.POISSON3, 4)
    D = bsr_dense(p, c, v)
    assert np.array_equal(D, D.T) and np.linalg.eigvalsh(D).min() > 0  # SPD (cfg 1)


def test_rng_moments():
    z = np.array([gen.n01(5, i) for i in range(20000)])
    assert abs(z.mean()) < 0.03 and abs(z.std() - 1) < 0.03
    u = np.array([gen.u01(2, i) for i in range(20000)])
    assert 0 <= u.min() and u.max() < 1 and abs(u.mean() - 0.5) < 0.01
