"""The CUDA ray cast can resume a walk mid-way (k_raycast_split, seek_prefix in
paper_2109_13176_b200/csrc/k_integrate.cu): the walk state after j0 steps is
found from the setup state alone.  Per axis it counts the crossings whose
stateless key lies below a threshold K chosen a few steps short of j0 (a float
guess corrected to the exact count with the keys, which are monotone per
axis), then takes the remaining j0 - sum(c) events with the exact step rule.
The events below any threshold form a prefix of the walk's (key, axis) order,
so the resumed walk is the original walk from step j0 on.  This test restates
that rule in numpy float32 and checks it against the oracle's walk
(or_traverse) at many j0 of random rays; the GPU parity tests check the
kernel."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.test_dda_fastpath_rule import INF, _count_before, _key, f32


def setup(dims, s, g):
    """The kernel's setup: per-axis (e1, f, inv, jmax) and the walk length T;
    None for its slow path."""
    S = [int(np.floor(s[a])) for a in range(3)]
    E = [int(np.floor(g[a])) for a in range(3)]
    st, rem, room = [0] * 3, [0] * 3, [0] * 3
    e1, f, inv, jmax = [f32(0)] * 3, [f32(0)] * 3, [INF] * 3, [0] * 3
    for a in range(3):
        st[a] = (E[a] > S[a]) - (E[a] < S[a])
        rem[a] = abs(E[a] - S[a])
        room[a] = (dims[a] - 1 - S[a]) if st[a] > 0 else S[a]
        f[a] = f32(st[a])
        e1[a] = f32(S[a] + (1 if st[a] >= 0 else 0))
        if rem[a] > 0:
            with np.errstate(all="ignore"):
                inv[a] = f32(1) / f32(g[a] - s[a])
            if not np.isfinite(inv[a]):
                return None
            jmax[a] = min(rem[a], room[a] + 1)
    exits = [a for a in range(3) if rem[a] > room[a]]
    if exits:
        Ka, aa = min((_key(e1[a], f[a], s[a], inv[a], room[a] + 1), a) for a in exits)
        T = room[aa] + 1
        for b in range(3):
            if b != aa and rem[b] > 0:
                T += _count_before(e1[b], f[b], s[b], inv[b], jmax[b], Ka, b < aa)
    else:
        T = sum(rem)
    return S, st, e1, f, inv, jmax, T


def seek_prefix(e1, f, s, inv, jmax, j0):
    """Kernel rule: (c[3], forward steps) for the state after j0 steps."""
    dabs = [abs(f32(1) / inv[a]) if jmax[a] > 0 else f32(0) for a in range(3)]
    Rm = f32(sum(dabs))
    K = f32(f32(j0 - 3.5) / Rm)
    for it in range(64):
        c = [0, 0, 0]
        for a in range(3):
            if jmax[a] > 0 and K > 0:
                X = f32(K * dabs[a] - f[a] * f32(e1[a] - s[a]) + 1)
                ca = int(np.ceil(X)) - 1
                ca = min(max(ca, 0), jmax[a])
                while ca < jmax[a] and _key(e1[a], f[a], s[a], inv[a], ca + 1) < K:
                    ca += 1
                while ca > 0 and not _key(e1[a], f[a], s[a], inv[a], ca) < K:
                    ca -= 1
                c[a] = ca
        if sum(c) <= j0:
            return c, j0 - sum(c)
        K = f32(K - f32(sum(c) - j0 + 2) / Rm) if it < 4 else f32(-1)
    raise AssertionError("no prefix")


def resumed_walk(dims, s, g, j0):
    r = setup(dims, s, g)
    if r is None:
        return None, None
    S, st, e1, f, inv, jmax, T = r
    if j0 >= T:
        return [], 0
    c, nf = seek_prefix(e1, f, s, inv, jmax, j0)
    e = [f32(e1[a] + f[a] * c[a]) for a in range(3)]
    with np.errstate(all="ignore"):
        k = [f32(f32(e[a] - s[a]) * inv[a]) if jmax[a] > 0 else INF for a in range(3)]
    V = [S[a] + st[a] * c[a] for a in range(3)]
    walk = []
    for step in range(T - j0 + nf):
        if step >= nf:
            walk.append(tuple(V))
        l10 = k[1] < k[0]
        b01 = k[1] if l10 else k[0]
        u2 = k[2] < b01
        a = 2 if u2 else (1 if l10 else 0)
        e[a] = f32(e[a] + f[a])
        V[a] += st[a]
        with np.errstate(all="ignore"):
            k[a] = f32(f32(e[a] - s[a]) * inv[a])
    return walk, nf


@pytest.mark.parametrize("seed", [0, 1])
def test_resumed_walk_equals_oracle_suffix(seed):
    rs = np.random.default_rng(100 + seed)
    checked = 0
    nfs = []
    for it in range(400):
        dims = (int(rs.integers(1, 90)), int(rs.integers(1, 90)), int(rs.integers(1, 30)))
        s = np.array([rs.uniform(0, dims[a]) for a in range(3)], dtype=np.float32)
        if it % 3 == 0:
            s = np.floor(s).astype(np.float32)  # sensor on integer planes
        g = (s + rs.normal(0, 60, size=3)).astype(np.float32)
        if it % 4 == 0:
            g = (np.round(g * 2) / 2).astype(np.float32)  # endpoints on half-planes
        if it % 7 == 0:
            g[rs.integers(0, 3)] = s[rs.integers(0, 3)]  # rays in grid planes
        ref = [tuple(v) for v in O.traverse(dims, s, g).tolist()]
        for j0 in sorted(set([1, 2, 3, 5, 32, 64] + list(rs.integers(1, max(2, len(ref) + 2), 6)))):
            got, nf = resumed_walk(dims, s, g, int(j0))
            if got is None:
                break  # slow path: the kernel walks such rays whole (half 0)
            assert got == ref[j0:], (dims, s.tolist(), g.tolist(), j0)
            if got:
                nfs.append(nf)
                checked += 1
    assert checked > 800
    # the guess lands a few events short of j0: the exact steps it leaves are few
    assert max(nfs) <= 8 and float(np.mean(nfs)) < 4.5, (max(nfs), np.mean(nfs))


def test_resume_on_lidar_rays():
    from paper_2109_13176_b200 import synth
    w = synth.workload(1)
    f = w.frames[0]
    sc = f.scans[0]
    o = O.snap_origin(256, 256, 64, 0.25, 0.5, f.vehicle_xyz)
    A, b = O.affine(sc.pose, 0.25, o)
    rs = np.random.default_rng(3)
    for i in rs.choice(sc.points.shape[0], 300, replace=False):
        ok, gg = O.transform_point(A, b, *sc.points[i, :3])
        ref = [tuple(v) for v in O.traverse((256, 256, 64), b, gg).tolist()]
        for j0 in (64, 128, 192):
            got, _ = resumed_walk((256, 256, 64), b, gg, j0)
            if got is None:
                break
            assert got == ref[j0:]
