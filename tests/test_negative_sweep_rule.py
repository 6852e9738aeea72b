"""The CUDA negative-obstacle kernel does not probe rings cell by cell as the
oracle's O10 does: it sweeps each cone direction with the recurrence
  D(x,y) = 1 if ring 1 holds a defined cell, else 1 + min_t D(x+1, y+t),
carrying the min / max heights of the first non-empty ring, with apexes up to
K cells outside the map, and decides max - min > T_neg (T_neg >= 0 makes the
oracle's |F| >= 2 implied).  See k_negative in csrc/k_maps.cu.  This test
re-states the sweep in plain Python and checks it against the oracle
(or_negative) on random height maps, including map edges, sparse and dense
defined masks and K larger than the map."""
import numpy as np
import pytest

from oracle import oracle as O

UNDEF = None


def sweep_negative(qs, defined, K, T_neg):
    ny, nx = qs.shape
    nmin = np.full((ny, nx), np.iinfo(np.int64).max, dtype=np.int64)
    nmax = np.full((ny, nx), np.iinfo(np.int64).min, dtype=np.int64)
    INF = K + 1
    for cone in range(4):
        alongx = cone < 2
        dirn = -1 if cone & 1 else 1
        A, B = (nx, ny) if alongx else (ny, nx)

        def q_at(p, b):  # line p, cross b
            if not (0 <= p < A and 0 <= b < B):
                return None
            y, x = (b, p) if alongx else (p, b)
            return int(qs[y, x]) if defined[y, x] else None

        prev = {b: (INF, None, None) for b in range(-K - 1, B + K + 1)}
        order = range(A - 1, -1, -1) if dirn > 0 else range(0, A)
        for p in order:
            cur = {}
            for b in range(-K, B + K):
                Dv, mn, mx = INF, None, None
                ring1 = [q for t in (-1, 0, 1) for q in [q_at(p + dirn, b + t)] if q is not None]
                if ring1:
                    Dv, mn, mx = 1, min(ring1), max(ring1)
                else:
                    subs = [prev.get(b + t, (INF, None, None)) for t in (-1, 0, 1)]
                    dm = min(s[0] for s in subs)
                    if dm < K:
                        Dv = dm + 1
                        mn = min(s[1] for s in subs if s[0] == dm)
                        mx = max(s[2] for s in subs if s[0] == dm)
                cur[b] = (Dv, mn, mx)
                if Dv <= K and 0 <= b < B:
                    y, x = (b, p) if alongx else (p, b)
                    nmin[y, x] = min(nmin[y, x], mn)
                    nmax[y, x] = max(nmax[y, x], mx)
            prev = cur
    neg = np.zeros((ny, nx), np.uint8)
    found = nmax != np.iinfo(np.int64).min
    neg[(defined == 0) & found & ((nmax - nmin) > T_neg)] = 1
    return neg


@pytest.mark.parametrize("seed,shape,density,K", [
    (0, (9, 11), 0.15, 3), (1, (12, 7), 0.05, 5), (2, (10, 10), 0.5, 2),
    (3, (6, 14), 0.02, 20), (4, (13, 13), 0.3, 6)])
def test_sweep_equals_oracle_cone_search(seed, shape, density, K):
    rs = np.random.default_rng(seed)
    for trial in range(6):
        defined = (rs.random(shape) < density).astype(np.uint8)
        qs = rs.integers(-300000, 300000, size=shape).astype(np.int32)
        T = int(rs.choice([0, 50000, 131072, 400000]))
        ref = O.negative(qs, defined, K, T)
        got = sweep_negative(qs, defined, K, T)
        assert np.array_equal(got, ref), (seed, trial)
