"""The CUDA ray-cast kernel does not run the oracle's O5 loop verbatim (see
k_raycast in paper_2109_13176_b200/csrc/k_integrate.cu):

* it keeps float edges e_a = f32(V_a + [step>0]) (exact small integers) and
  recomputes key_a = f32(f32(e_a - s_a) * inv_a) from them;
* it computes the walk length T at setup: with no grid exit, T = sum rem_a;
  otherwise the first exit crossing (key, axis) = min over exit axes a of
  key_a(room_a + 1) and T = 1 + room_a* + the number of other-axis crossings
  that precede it in (key, axis) order (binary search: keys are monotone);
* it then runs T steps of a plain argmin (strict <, ties to the lowest axis)
  with no per-step gating, after checking once that no exhausted axis's next
  ("overshoot") key could precede the walk's last crossing; rays failing that
  check, or with a non-finite reciprocal, take an exact slow path.

This test restates that rule in numpy float32 and checks it step for step
against the oracle's walk (or_traverse) on random rays, including sensors on
integer planes, endpoints on half-integers and rays in grid planes; it also
reports how often the slow path is taken.  The GPU parity tests check the
kernel itself."""
import numpy as np
import pytest

from oracle import oracle as O

f32 = np.float32
INF = f32(np.inf)


def _key(e1, f, s, inv, j):
    # key of the j-th crossing (j >= 1) on an axis
    with np.errstate(all="ignore"):
        return f32(f32(f32(e1 + f32(f * (j - 1))) - s) * inv)


def _count_before(e1, f, s, inv, jmax, K, tie_ok):
    lo, hi = 0, jmax
    while lo < hi:
        mid = (lo + hi + 1) // 2
        k = _key(e1, f, s, inv, mid)
        if k < K or (k == K and tie_ok):
            lo = mid
        else:
            hi = mid - 1
    return lo


def walk_fastpath(dims, s, g):
    """Returns the walk, or None when the kernel would take its slow path."""
    S = [int(np.floor(s[a])) for a in range(3)]
    E = [int(np.floor(g[a])) for a in range(3)]
    st, rem, room, e1, f, inv = [0] * 3, [0] * 3, [0] * 3, [f32(0)] * 3, [f32(0)] * 3, [INF] * 3
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
    exits = [a for a in range(3) if rem[a] > room[a]]
    if exits:
        Ka, aa = min((_key(e1[a], f[a], s[a], inv[a], room[a] + 1), a) for a in exits)
        T = room[aa] + 1  # emits: the start voxel + every crossing before the exit
        for b in range(3):
            if b != aa and rem[b] > 0:
                jmax = min(rem[b], room[b] + 1)
                T += _count_before(e1[b], f[b], s[b], inv[b], jmax, Ka, b < aa)
        end = (Ka, aa)  # every walk crossing precedes the exit crossing
    else:
        T = sum(rem)
        last = [(_key(e1[b], f[b], s[b], inv[b], rem[b]), b) for b in range(3) if rem[b] > 0]
        end = max(last) if last else None
    # an exhausted (non-exit) axis must never be the argmin before the end
    for a in range(3):
        if rem[a] > 0 and a not in exits and end is not None:
            ov = (_key(e1[a], f[a], s[a], inv[a], rem[a] + 1), a)
            if not ov > end:
                return None
    e = list(e1)
    k = [(_key(e1[a], f[a], s[a], inv[a], 1) if rem[a] > 0 else INF) for a in range(3)]
    V = list(S)
    walk = []
    for _ in range(T):
        walk.append(tuple(V))
        l10 = k[1] < k[0]
        b01 = k[1] if l10 else k[0]
        u2 = k[2] < b01
        a = 2 if u2 else (1 if l10 else 0)
        e[a] = f32(e[a] + f[a])
        V[a] += st[a]
        with np.errstate(all="ignore"):
            k[a] = f32(f32(e[a] - s[a]) * inv[a])
    return walk


@pytest.mark.parametrize("seed", [0, 1])
def test_fastpath_rule_equals_oracle_walk(seed):
    rs = np.random.default_rng(seed)
    checked = slow = 0
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
            g[rs.integers(0, 3)] = s[rs.integers(0, 3)]  # rays in grid planes
        got = walk_fastpath(dims, s, g)
        if got is None:
            slow += 1
            continue
        ref = [tuple(v) for v in O.traverse(dims, s, g).tolist()]
        assert got == ref, (dims, s.tolist(), g.tolist())
        checked += 1
    assert checked > 2300, (checked, slow)


def test_fastpath_slow_path_is_rare_on_lidar_rays():
    from paper_2109_13176_b200 import synth
    w = synth.workload(1)
    f = w.frames[0]
    s = f.scans[0]
    o = O.snap_origin(256, 256, 64, 0.25, 0.5, f.vehicle_xyz)
    A, b = O.affine(s.pose, 0.25, o)
    rs = np.random.default_rng(0)
    idx = rs.choice(s.points.shape[0], 3000, replace=False)
    slow = 0
    for i in idx:
        ok, gg = O.transform_point(A, b, *s.points[i, :3])
        got = walk_fastpath((256, 256, 64), b, gg)
        if got is None:
            slow += 1
            continue
        assert got == [tuple(v) for v in O.traverse((256, 256, 64), b, gg).tolist()]
    assert slow <= 3
