"""The CUDA ray-cast kernel does not run the oracle's O5 loop verbatim: it
keeps float edges instead of recomputing f32(V + [step>0]), gives exhausted
axes a +inf key (1/d := +-inf) instead of gating on rem > 0, and ends a walk
through precomputed per-axis room counters instead of a bounds test (see
paper_2109_13176_b200/csrc/k_integrate.cu, k_raycast).  This test re-states
that rule step for step in numpy float32 and checks it against the oracle's
walk (oracle/gvom_oracle.c or_traverse) on random rays, including sensors on
integer planes, endpoints on half-integers and rays along grid planes -- the
argument for why the kernel is bit-exact, checked on the CPU.  The GPU parity
tests check the kernel itself."""
import numpy as np
import pytest

from oracle import oracle as O

f32 = np.float32
INF = f32(np.inf)


def walk_fastpath(dims, s, g):
    n = dims
    S = [int(np.floor(s[a])) for a in range(3)]
    E = [int(np.floor(g[a])) for a in range(3)]
    e, f, inv, k, c, x, r = [0] * 3, [0] * 3, [INF] * 3, [INF] * 3, [0] * 3, [False] * 3, [0] * 3
    for a in range(3):
        st = (E[a] > S[a]) - (E[a] < S[a])
        r[a] = abs(E[a] - S[a])
        room = (n[a] - 1 - S[a]) if st > 0 else S[a]
        f[a] = f32(st)
        e[a] = f32(S[a] + (1 if st >= 0 else 0))
        x[a] = r[a] > room
        c[a] = room if x[a] else r[a]
        if r[a] > 0:
            with np.errstate(all="ignore"):
                inv[a] = f32(1) / f32(g[a] - s[a])
                k[a] = f32(f32(e[a] - s[a]) * inv[a])
            if not np.isfinite(inv[a]):
                return None  # the kernel's exact slow path
    V = list(S)
    walk = []
    left = sum(n) if any(x) else sum(r)
    active = sum(r) > 0
    while active:
        walk.append(tuple(V))
        l10 = k[1] < k[0]
        b01 = k[1] if l10 else k[0]
        u2 = k[2] < b01
        u1 = l10 and not u2
        a = 2 if u2 else (1 if u1 else 0)
        cs, xs = c[a], x[a]
        out = xs and cs == 0
        e[a] = f32(e[a] + f[a])
        c[a] -= 1
        V[a] += int(f[a])
        if (not xs) and cs == 1:
            inv[a] = f32(f[a] * INF)
        with np.errstate(all="ignore"):
            for b in range(3):
                k[b] = f32(f32(e[b] - s[b]) * inv[b])
        left -= 1
        active = active and not out and left != 0
    return walk


@pytest.mark.parametrize("seed", [0, 1])
def test_fastpath_rule_equals_oracle_walk(seed):
    rs = np.random.default_rng(seed)
    checked = 0
    for it in range(2500):
        dims = (int(rs.integers(1, 40)), int(rs.integers(1, 40)), int(rs.integers(1, 16)))
        s = np.array([rs.uniform(0, dims[a]) for a in range(3)], dtype=np.float32)
        if it % 3 == 0:
            s = np.floor(s).astype(np.float32)  # sensor on integer planes
        if it % 5 == 0:
            s[it % 3] = np.float32(0.0)
        g = (s + rs.normal(0, 25, size=3)).astype(np.float32)
        if it % 4 == 0:
            g = (np.round(g * 2) / 2).astype(np.float32)  # endpoints on half-planes
        if it % 7 == 0:
            g[rs.integers(0, 3)] = s[rs.integers(0, 3)]  # rays along grid planes
        got = walk_fastpath(dims, s, g)
        if got is None:
            continue
        ref = [tuple(v) for v in O.traverse(dims, s, g).tolist()]
        assert got == ref, (dims, s.tolist(), g.tolist())
        checked += 1
    assert checked > 2000
