// k_integrate.cu -- pointcloud processing (section III.C) on sm_100a.
//
//   raycast  : transform + endpoint occupancy bit + tile counts + float32 DDA
//              pass-through counts (the frame's last block scans the tile counts)
//   finalize : rank of occupied voxels in L order (from the tile offsets) +
//              in-place LUT encode (rank | -1 - N_m) + data rows; with
//              peer grids (NEXT-2) it sums the ranks' miss grids as it reads
//   rank     : single-pass rank over a bitmask (merged-map export path)
//   endpoint : per-return hits, lowest return, fixed-point moments into data rows
//
// Numerics: every float op that decides an integer is written as an explicit
// IEEE round-to-nearest intrinsic (__fmul_rn/__fadd_rn/__fsub_rn/__frcp_rn) in
// the order of SURVEY.md 8(c) O3/O5, and the file is built with -fmad=false, so
// the voxel walk is bit-identical to the oracle's.  Integer accumulation only
// (u32/u64 atomics): results are independent of thread schedule.
#include <cuda/atomic>
#include <stdlib.h>

#include "gvom_device.cuh"

namespace gvom {

namespace {

__device__ __forceinline__ int64_t point_index(int64_t tid, int32_t rings) {
  // Sensor-order scans (column-major, beam-fastest): lane l of a warp takes
  // column 32*tile + l of ring r, so a warp walks 32 azimuth-adjacent rays of
  // one ring in lockstep; rays that share a voxel reach it at the same step
  // (step index = Manhattan distance from the sensor voxel) and their miss
  // increments are merged before the atomic.  rings <= 1: identity.
  if (rings <= 1) return tid;
  const int64_t per_tile = 32 * (int64_t)rings;
  const int64_t tile = tid / per_tile;
  const int32_t w = (int32_t)(tid - tile * per_tile);
  const int32_t r = w >> 5;
  const int32_t l = w & 31;
  return (tile * 32 + l) * rings + r;
}

// Exact O5 walk of one ray, oracle control flow verbatim (slow path for the
// astronomically rare rays whose reciprocal 1/d_a is not finite, where the
// fast path's +inf-key gating would not be equivalent).
__device__ void walk_exact(const int S[3], const int E[3], const float g[3], const float s[3],
                           const Dims& d, uint32_t* __restrict__ miss, int y0, int y1,
                           uint32_t inc) {
  int V[3] = {S[0], S[1], S[2]}, st[3], rem[3];
  float inv[3];
  for (int a = 0; a < 3; ++a) {
    st[a] = (E[a] > S[a]) - (E[a] < S[a]);
    rem[a] = abs(E[a] - S[a]);
    inv[a] = rem[a] > 0 ? __frcp_rn(__fsub_rn(g[a], s[a])) : 0.0f;
  }
  const int n[3] = {d.nx, d.ny, d.nz};
  while ((unsigned)V[0] < (unsigned)n[0] && (unsigned)V[1] < (unsigned)n[1] &&
         (unsigned)V[2] < (unsigned)n[2] && rem[0] + rem[1] + rem[2] > 0) {
    if (V[1] >= y0 && V[1] < y1) atomicAdd(miss + (V[2] + d.nz * (V[0] + d.nx * V[1])), inc);
    int best = -1;
    float bk = 0.f;
    for (int a = 0; a < 3; ++a) {
      if (rem[a] <= 0) continue;
      const float key =
          __fmul_rn(__fsub_rn(__int2float_rn(V[a] + (st[a] > 0 ? 1 : 0)), s[a]), inv[a]);
      if (best < 0 || key < bk) {
        best = a;
        bk = key;
      }
    }
    V[best] += st[best];
    rem[best] -= 1;
  }
}

// key of the j-th crossing (j >= 1) of an axis: f32(f32(e_j - s) * inv) with
// the exact float edge e_j = e1 + step*(j-1)  (O5's stateless key)
__device__ __forceinline__ float axis_key(float e1, float f, float s, float inv, int j) {
  return __fmul_rn(__fsub_rn(__fadd_rn(e1, f * (float)(j - 1)), s), inv);
}

// number of crossings j in [1, jmax] of an axis that precede (K, tie_ok):
// key_j < K, or key_j == K with the axis ordered first.  Keys are monotone
// non-decreasing in j, so this is a binary search.
__device__ __forceinline__ int count_before(float e1, float f, float s, float inv, int jmax,
                                            float K, bool tie_ok) {
  int lo = 0, hi = jmax;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    const float k = axis_key(e1, f, s, inv, mid);
    if (k < K || (k == K && tie_ok))
      lo = mid;
    else
      hi = mid - 1;
  }
  return lo;
}

// (k, a) > (K, A) in the walk order (key, then axis index)
__device__ __forceinline__ bool after(float k, int a, float K, int A) {
  return k > K || (k == K && a > A);
}

// Ray cast (O5) for a frame's points.  The walk of a ray is the merge, in
// (key, axis) order, of its three monotone per-axis crossing sequences.  At
// setup each lane computes its exact walk length T (the emits: sum rem_a, or
// 1 + the crossings before the first grid-exit crossing, counted by binary
// search) and checks that no exhausted axis's next key can precede the
// walk's end; then it runs T ungated argmin steps.  Rays failing the check or
// with a non-finite 1/d take the exact slow path.  The rule is restated and
// checked against the oracle in tests/test_dda_fastpath_rule.py.

// The frame's last finishing ray-cast block (of the last sensor's launch)
// turns the tile counts into exclusive offsets: each thread sums a
// contiguous chunk, one block scan of the chunk sums, then each thread
// writes its chunk's running offsets.
__device__ void scan_tiles_if_last(const TileCounts& tc, const Dims& d) {
  __shared__ bool last;
  __shared__ uint32_t wsum[32];
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(tc.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t nt = n_tiles(d);
  const int64_t chunk = (nt + blockDim.x - 1) / blockDim.x;
  const int64_t c0 = threadIdx.x * chunk, c1 = min(nt, c0 + chunk);
  uint32_t sum = 0;
  for (int64_t i = c0; i < c1; ++i) sum += __ldcg(tc.tile + i);
  const uint32_t inc = warp_incl_scan(sum, lane);
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const uint32_t w = lane < nw ? wsum[lane] : 0u;
    const uint32_t e = warp_incl_scan(w, lane) - w;
    if (lane < nw) wsum[lane] = e;
  }
  __syncthreads();
  uint32_t run = wsum[wid] + inc - sum;
  for (int64_t i = c0; i < c1; ++i) {
    tc.offset[i] = run;
    run += __ldcg(tc.tile + i);
  }
  if (threadIdx.x == 0) *tc.done = 0u;  // every block has counted: ready for the next frame
}

// Miss increments of one warp step, merged over runs of adjacent lanes that
// hold the same voxel: one red.add per run, issued by its first lane.  Two
// schedules, chosen per launch by the miss grid's size (launch_raycast):
//  - resident (kStream = false; the grid fits in L2): L is a 32-bit BYTE offset
//    and an inactive lane carries the key ~0, which breaks runs by itself, so
//    the step needs no mask of active lanes and runs on a warp-uniform trip
//    count (fewest instructions per step);
//  - streaming (kStream = true; REDs go out to HBM): L is the voxel index and
//    the run count masks the inactive lanes; this schedule measured faster
//    when the REDs are DRAM-latency bound (c5: 2.88 vs 3.08 ms), the resident
//    one faster when they hit L2 (c2: 50 vs 55 us) -- see DESIGN.md.
template <bool kStream>
__device__ __forceinline__ uint32_t* miss_at(uint32_t* miss, uint32_t L) {
  if (kStream) return miss + L;
  return reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(miss) + L);
}

__device__ __forceinline__ void red_run(uint32_t* addr, bool head, uint32_t cnt) {
  // no "memory" clobber: nothing in the kernel reads the miss grid, so the
  // reduction needs no ordering with the surrounding code
  asm volatile(
      "{ .reg .pred p; setp.ne.u32 p, %2, 0;\n\t"
      "@p red.relaxed.gpu.global.add.u32 [%0], %1; }" ::"l"(addr),
      "r"(cnt), "r"((uint32_t)head));
}

// resident schedule: see above.  kNeg: the run adds -count (the integrate
// path counts misses down from -1 directly in the LUT: -1 - N_m, O6)
template <bool kNeg>
__device__ __forceinline__ void aggregate_red_resident(uint32_t* __restrict__ miss, uint32_t L,
                                                       bool active, bool lane0,
                                                       unsigned after_lanes, int lane) {
  const uint32_t key = active ? L : 0xffffffffu;
  const uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
  const bool brk = prev != key;
  const unsigned heads = __ballot_sync(0xffffffffu, brk);
  const bool head = active && (brk || lane0);
  // run length = distance to the next run start above this lane (32 if none):
  // ctz(x) = popc(~x & (x - 1)), which is 32 for x = 0 without a special case
  if (kNeg)
    asm volatile(
        "{ .reg .pred p; .reg .b32 t, u;\n\t"
        "and.b32 t, %1, %2;\n\t"
        "add.u32 u, t, -1;\n\t"
        "not.b32 t, t;\n\t"
        "and.b32 t, t, u;\n\t"
        "popc.b32 t, t;\n\t"
        "sub.u32 t, %3, t;\n\t"
        "setp.ne.u32 p, %4, 0;\n\t"
        "@p red.relaxed.gpu.global.add.u32 [%0], t; }" ::"l"(miss_at<false>(miss, L)),
        "r"(heads), "r"(after_lanes), "r"(lane), "r"((uint32_t)head));
  else
    asm volatile(
        "{ .reg .pred p; .reg .b32 t, u;\n\t"
        "and.b32 t, %1, %2;\n\t"
        "add.u32 u, t, -1;\n\t"
        "not.b32 t, t;\n\t"
        "and.b32 t, t, u;\n\t"
        "popc.b32 t, t;\n\t"
        "sub.u32 t, t, %3;\n\t"
        "setp.ne.u32 p, %4, 0;\n\t"
        "@p red.relaxed.gpu.global.add.u32 [%0], t; }" ::"l"(miss_at<false>(miss, L)),
        "r"(heads), "r"(after_lanes), "r"(lane), "r"((uint32_t)head));
}

// streaming schedule: `act` = the warp's active lanes
template <bool kNeg>
__device__ __forceinline__ void aggregate_red_stream(uint32_t* __restrict__ miss, uint32_t L,
                                                     bool active, unsigned act,
                                                     unsigned after_lanes, int lane) {
  const uint32_t key = active ? L : 0xffffffffu;
  const uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
  const bool head = active && (lane == 0 || prev != key);
  const unsigned heads = __ballot_sync(0xffffffffu, head);
  const int run = __clz(__brev((heads | ~act) & after_lanes)) - lane;
  red_run(miss_at<true>(miss, L), head, kNeg ? (uint32_t)(-run) : (uint32_t)run);
}

#ifndef GVOM_RAY_STREAM_BYTES
#define GVOM_RAY_STREAM_BYTES 0
#endif
// miss grids above half the L2 (B200: 126 MB split over two dies, so 64 MB;
// tuned on c4 / c5) take the streaming schedule; a nonzero
// GVOM_RAY_STREAM_BYTES overrides the threshold (A/B builds)
constexpr int64_t kRayStreamBytes = GVOM_RAY_STREAM_BYTES;

// One DDA step (O5): argmin of the three keys, strict <, ties to the lowest
// axis; no gating needed: a lane past its walk keeps stepping unseen (its
// exhausted axes carry +inf keys, see the setup in k_raycast).
__device__ __forceinline__ void dda_step(float& k0, float& k1, float& k2, float& e0, float& e1,
                                         float& e2, float f0, float f1, float f2, float i0,
                                         float i1, float i2, float s0, float s1, float s2,
                                         int dL0, int dL1, int dL2, uint32_t& L) {
  const bool l10 = k1 < k0;
  const float b01 = l10 ? k1 : k0;
  const bool u2 = k2 < b01;
  const bool u1 = l10 && !u2;
  const bool u0 = !l10 && !u2;
  e0 = u0 ? __fadd_rn(e0, f0) : e0;
  e1 = u1 ? __fadd_rn(e1, f1) : e1;
  e2 = u2 ? __fadd_rn(e2, f2) : e2;
  L += (uint32_t)(u2 ? dL2 : (u1 ? dL1 : dL0));
  k0 = __fmul_rn(__fsub_rn(e0, s0), i0);
  k1 = __fmul_rn(__fsub_rn(e1, s1), i1);
  k2 = __fmul_rn(__fsub_rn(e2, s2), i2);
}

#ifndef GVOM_RESET_V8
#define GVOM_RESET_V8 1  // k_reset_slot with 32-byte stores (A/B builds: 0 = 16-byte)
#endif
#ifndef GVOM_RAY_STREAM_PREFIX
#define GVOM_RAY_STREAM_PREFIX 1
#endif
#ifndef GVOM_RAY_UNROLL
#define GVOM_RAY_UNROLL 1
#endif
constexpr int kRayUnroll = GVOM_RAY_UNROLL;
// The step loop of a warp: one aggregated red per step, then one DDA step.
template <bool kStream, bool kNeg, class Step>
__device__ __forceinline__ void walk_loop(uint32_t* __restrict__ miss, const uint32_t& L, int left,
                                          int lane, unsigned after_lanes, Step&& step) {
  if (kStream) {
    // the first Tmin steps have every lane active: no per-step ballot
    // (GVOM_RAY_STREAM_PREFIX=0: without this prefix, A/B builds)
#if GVOM_RAY_STREAM_PREFIX
    const int Tmin = __reduce_min_sync(0xffffffffu, left);
    for (int it = 0; it < Tmin; ++it) {
      aggregate_red_stream<kNeg>(miss, L, true, 0xffffffffu, after_lanes, lane);
      step();
    }
    left -= Tmin;
#endif
    unsigned act = __ballot_sync(0xffffffffu, left > 0);
    while (act) {
      const bool active = left > 0;
      aggregate_red_stream<kNeg>(miss, L, active, act, after_lanes, lane);
      step();
      --left;
      act = __ballot_sync(0xffffffffu, left > 0);
    }
  } else {
    const bool lane0 = lane == 0;
    // warp-uniform trip count: lane i is active for its first left_i steps;
    // the first Tmin steps have every lane active (71 % of the c2 warp-steps),
    // so they skip the per-step activity test (c2 ray cast 48.0 vs 49.6 us,
    // c3 70.0 vs 72.5 us, c4 tie)
    const int Tw = __reduce_max_sync(0xffffffffu, left);
    const int Tmin = __reduce_min_sync(0xffffffffu, left);
    int it = 0;
#pragma unroll (kRayUnroll)
    for (; it < Tmin; ++it) {
      aggregate_red_resident<kNeg>(miss, L, true, lane0, after_lanes, lane);
      step();
    }
#pragma unroll (kRayUnroll)
    for (; it < Tw; ++it) {
      const bool active = it < left;
      aggregate_red_resident<kNeg>(miss, L, active, lane0, after_lanes, lane);
      step();
    }
  }
}

// The step loop of a warp whose lanes walk steps [start_i, end_i) of their
// rays (the ray-segment slab partition): iterations run over absolute step
// indices, so lanes that reach a voxel at the same step still merge; a lane
// holds its state until its start.
template <bool kStream, bool kNeg, class Step>
__device__ __forceinline__ void walk_loop_range(uint32_t* __restrict__ miss, const uint32_t& L,
                                                int start, int end, int lane,
                                                unsigned after_lanes, Step&& step) {
  const bool has = start < end;
  const int w0 = __reduce_min_sync(0xffffffffu, has ? start : 0x7fffffff);
  const int w1 = __reduce_max_sync(0xffffffffu, has ? end : 0);
  const bool lane0 = lane == 0;
  for (int it = w0; it < w1; ++it) {
    const bool active = it >= start && it < end;
    if (kStream)
      aggregate_red_stream<kNeg>(miss, L, active, __ballot_sync(0xffffffffu, active),
                                 after_lanes, lane);
    else
      aggregate_red_resident<kNeg>(miss, L, active, lane0, after_lanes, lane);
    if (it >= start) step();
  }
}

// Steps taken once the walk has taken its c-th crossing of the y axis (axis 1):
// that crossing, the c - 1 before it, and the x / z crossings that precede it in
// the walk's (key, axis) order (x first on equal keys, z after) -- the index of
// the first voxel of the walk beyond that y plane.  cnt[] = the crossings per axis.
__device__ __forceinline__ int steps_through_y(const float eb[3], const float fb[3],
                                               const float s[3], const float inv[3],
                                               const int jm[3], int c, int cnt[3]) {
  const float K = axis_key(eb[1], fb[1], s[1], inv[1], c);
  cnt[0] = jm[0] > 0 ? count_before(eb[0], fb[0], s[0], inv[0], jm[0], K, true) : 0;
  cnt[1] = c;
  cnt[2] = jm[2] > 0 ? count_before(eb[2], fb[2], s[2], inv[2], jm[2], K, false) : 0;
  return cnt[0] + c + cnt[2];
}

// State after the first j0 steps of a walk (kSplit's second half): c[a] = the
// axis-a crossings among the walk's first j0 events.  The events (key, axis)
// with key < K form a prefix of the walk's (key, axis) order for any
// threshold K, so counting the crossings below a K chosen a few steps short of
// j0 (K * sum |d_a| ~ j0 - 3.5) gives a prefix of j <= j0 events; the caller
// takes the j0 - j remaining events with the exact step rule.  Each count is a
// float guess corrected to the exact count with the stateless keys (monotone
// in j).  j0 < T, so no exhausted axis's key is below K.  Returns j0 - j.
__device__ __forceinline__ int seek_prefix(const float eb[3], const float fb[3], const float s[3],
                                           const float inv[3], const int jmax[3], int j0,
                                           int c[3]) {
  float dabs[3], Rm = 0.f;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    dabs[a] = jmax[a] > 0 ? fabsf(__fdividef(1.0f, inv[a])) : 0.f;
    Rm += dabs[a];
  }
  float K = __fdividef((float)j0 - 3.5f, Rm);
  for (int iter = 0;; ++iter) {
    int sum = 0;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      int ca = 0;
      if (jmax[a] > 0 && K > 0.f) {
        const float X = K * dabs[a] - fb[a] * (eb[a] - s[a]) + 1.0f;
        ca = (int)ceilf(X) - 1;
        ca = ca < 0 ? 0 : (ca > jmax[a] ? jmax[a] : ca);
        while (ca < jmax[a] && axis_key(eb[a], fb[a], s[a], inv[a], ca + 1) < K) ++ca;
        while (ca > 0 && !(axis_key(eb[a], fb[a], s[a], inv[a], ca) < K)) --ca;
      }
      c[a] = ca;
      sum += ca;
    }
    if (sum <= j0) return j0 - sum;
    // overshoot (float guess of K): retreat; after a few tries start from 0
    K = iter < 4 ? K - __fdividef((float)(sum - j0) + 2.0f, Rm) : -1.0f;
  }
}

// The rays of one warp (32 consecutive thread ids gtid of the batch).
// kSplit (A/B: GVOM_RAY_SPLIT=1): two warps per 32 rays, half 0 walking the
// first ceil(Tw / 2) steps and half 1 the rest from the exact state at that
// step (seek_prefix + the exact step rule), so a block's critical path is half
// the longest walk; only half 0 bins the endpoints.
// kSlab: only the steps whose voxel lies in rows [sr.y0, sr.y1) are traced and
// only returns in those rows are binned (y is monotone along a walk, so that
// is one step range [jin, jout), found exactly with the stateless keys).
template <bool kStream, bool kNeg, bool kSlab = false, bool kSplit = false>
__device__ __forceinline__ void ray_warp(const RayBatch& rb, const Dims& d,
                                         uint32_t* __restrict__ miss, uint32_t* __restrict__ bits,
                                         const TileCounts& tc, int64_t gtid,
                                         const SlabRange sr = SlabRange{0, 0}, int half = 0) {
  const int64_t gt = gtid / rb.tile_threads;  // interleaved (tile, sensor)
  const int sidx = (int)(gt % rb.S);
  const int64_t tid = (gt / rb.S) * rb.tile_threads + (gtid - gt * rb.tile_threads);
  const int rings = rb.rings;
  const int64_t n = rb.n[sidx];
  const float4* __restrict__ pts = rb.pts[sidx];
  const SensorParams sp = rb.sp[sidx];
  const int64_t p = point_index(tid, rings);
  const int lane = threadIdx.x & 31;
  const float s0 = sp.b[0], s1 = sp.b[1], s2 = sp.b[2];
  const float kInf = __int_as_float(0x7f800000);

  float e0 = 0.f, e1 = 0.f, e2 = 0.f, f0 = 0.f, f1 = 0.f, f2 = 0.f;
  float i0 = kInf, i1 = kInf, i2 = kInf, k0 = kInf, k1 = kInf, k2 = kInf;
  int dL0 = 0, dL1 = 0, dL2 = 0, left = 0;
  int jm0 = 0, jm1 = 0, jm2 = 0;  // crossings each axis can take (kSlab)
  int jin = 0;                    // kSlab: first step in the slab (left = its end)
  uint32_t L = 0;
  uint32_t newtile = 0xffffffffu;  // tile of a voxel this lane newly occupied

  if (p < n) {
    const float4 qp = __ldg(pts + p);
    float g[3];
    if (transform_point(sp, qp, g[0], g[1], g[2])) {
      const int n3[3] = {d.nx, d.ny, d.nz};
      const int strideY = d.nz * d.nx;
      const int str[3] = {d.nz, strideY, 1};
      const float s[3] = {s0, s1, s2};
      int E[3], st[3], rem[3], room[3];
      float eb[3], fb[3], inv[3];
      bool fin = true;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        E[a] = (int)floorf(g[a]);
        st[a] = (E[a] > sp.S[a]) - (E[a] < sp.S[a]);
        rem[a] = abs(E[a] - sp.S[a]);
        room[a] = st[a] > 0 ? (n3[a] - 1 - sp.S[a]) : sp.S[a];
        fb[a] = (float)st[a];
        eb[a] = (float)(sp.S[a] + (st[a] >= 0 ? 1 : 0));
        inv[a] = kInf;
        if (rem[a] > 0) {
          inv[a] = __frcp_rn(__fsub_rn(g[a], s[a]));
          fin = fin && isfinite(inv[a]);
        }
      }
      // endpoint occupancy (O4/O6: occupied iff hits >= 1); bits == nullptr in
      // the multi-GPU partial pass (occupancy is built on the slab owner)
      if (bits && (!kSplit || half == 0) && (unsigned)E[0] < (unsigned)d.nx &&
          (unsigned)E[1] < (unsigned)d.ny && (unsigned)E[2] < (unsigned)d.nz &&
          (!kSlab || (E[1] >= sr.y0 && E[1] < sr.y1))) {
        const uint32_t LE = (uint32_t)(E[2] + d.nz * E[0] + strideY * E[1]);
        const uint32_t bit = 1u << (LE & 31);
        newtile = (atomicOr(bits + (LE >> 5), bit) & bit) ? 0xffffffffu : (LE >> kTileShift);
      }
      const int R = rem[0] + rem[1] + rem[2];
      // kSlab: a segment whose rows [min(S_y, E_y), max(S_y, E_y)] miss the slab
      // has no step there -- skip its setup (most rays of an outer slab)
      const bool miss_slab =
          kSlab && (max(sp.S[1], E[1]) < sr.y0 || min(sp.S[1], E[1]) >= sr.y1);
      if (R > 0 && !miss_slab) {
        bool ok = fin;
        float Kend = 0.f;
        int Aend = -1;
        bool anyexit = false;
        if (ok) {
          // first exit crossing (key, axis)
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            if (rem[a] > room[a]) {
              const float kx = axis_key(eb[a], fb[a], s[a], inv[a], room[a] + 1);
              if (!anyexit || kx < Kend) {
                Kend = kx;
                Aend = a;
              }
              anyexit = true;
            }
          }
          if (anyexit) {
            int T = 1;
#pragma unroll
            for (int b = 0; b < 3; ++b) {
              if (b == Aend)
                T += room[b];
              else if (rem[b] > 0)
                T += count_before(eb[b], fb[b], s[b], inv[b], min(rem[b], room[b] + 1), Kend,
                                  b < Aend);
            }
            left = T;
          } else {
            left = R;
#pragma unroll
            for (int b = 0; b < 3; ++b) {
              if (rem[b] > 0) {
                const float kl = axis_key(eb[b], fb[b], s[b], inv[b], rem[b]);
                if (Aend < 0 || after(kl, b, Kend, Aend)) {
                  Kend = kl;
                  Aend = b;
                }
              }
            }
          }
          // no exhausted axis may become the argmin before the walk ends
#pragma unroll
          for (int a = 0; a < 3; ++a) {
            if (rem[a] > 0 && rem[a] <= room[a]) {
              const float ov = axis_key(eb[a], fb[a], s[a], inv[a], rem[a] + 1);
              ok = ok && after(ov, a, Kend, Aend);
            }
          }
        }
        if (!ok) {
          const int S[3] = {sp.S[0], sp.S[1], sp.S[2]};
          if (!kSplit || half == 0)
            walk_exact(S, E, g, s, d, miss, kSlab ? sr.y0 : 0, kSlab ? sr.y1 : d.ny,
                       kNeg ? 0xffffffffu : 1u);
          left = 0;
        } else {
          e0 = eb[0]; e1 = eb[1]; e2 = eb[2];
          f0 = fb[0]; f1 = fb[1]; f2 = fb[2];
          i0 = inv[0]; i1 = inv[1]; i2 = inv[2];
          k0 = rem[0] > 0 ? axis_key(eb[0], fb[0], s0, i0, 1) : kInf;
          k1 = rem[1] > 0 ? axis_key(eb[1], fb[1], s1, i1, 1) : kInf;
          k2 = rem[2] > 0 ? axis_key(eb[2], fb[2], s2, i2, 1) : kInf;
          constexpr int unit = kStream ? 1 : 4;  // see miss_at
          dL0 = st[0] * str[0] * unit;
          dL1 = st[1] * str[1] * unit;
          dL2 = st[2] * str[2] * unit;
          L = (uint32_t)(sp.S[2] + d.nz * sp.S[0] + strideY * sp.S[1]) * unit;
          jm0 = rem[0] > 0 ? min(rem[0], room[0] + 1) : 0;
          jm1 = rem[1] > 0 ? min(rem[1], room[1] + 1) : 0;
          jm2 = rem[2] > 0 ? min(rem[2], room[2] + 1) : 0;
          if (kSlab) {
            // [jin, jout): the steps whose voxel row lies in [y0, y1)
            const int Sy = sp.S[1];
            const int jm[3] = {jm0, jm1, jm2};
            int cnt[3] = {0, 0, 0};
            int jout = left;
            if (st[1] == 0) {
              if (Sy < sr.y0 || Sy >= sr.y1) jout = 0;
            } else {
              // y crossings to enter / to leave the slab (0: inside from the start)
              const int cin = st[1] > 0 ? (Sy < sr.y0 ? sr.y0 - Sy : 0)
                                        : (Sy >= sr.y1 ? Sy - (sr.y1 - 1) : 0);
              const bool before = st[1] > 0 ? Sy >= sr.y1 : Sy < sr.y0;  // already past
              const int cout = st[1] > 0 ? sr.y1 - Sy : Sy - sr.y0 + 1;
              if (before || cin > jm1) {
                jout = 0;
              } else {
                if (cout <= jm1) {
                  int c2[3];
                  jout = min(jout, steps_through_y(eb, fb, s, inv, jm, cout, c2));
                }
                if (cin > 0) jin = steps_through_y(eb, fb, s, inv, jm, cin, cnt);
              }
            }
            if (jin >= jout) {
              jin = jout = 0;
            } else if (jin > 0) {  // the walk's state at step jin
              e0 = __fadd_rn(eb[0], fb[0] * (float)cnt[0]);
              e1 = __fadd_rn(eb[1], fb[1] * (float)cnt[1]);
              e2 = __fadd_rn(eb[2], fb[2] * (float)cnt[2]);
              k0 = rem[0] > 0 ? __fmul_rn(__fsub_rn(e0, s0), i0) : kInf;
              k1 = rem[1] > 0 ? __fmul_rn(__fsub_rn(e1, s1), i1) : kInf;
              k2 = rem[2] > 0 ? __fmul_rn(__fsub_rn(e2, s2), i2) : kInf;
              L += (uint32_t)(cnt[0] * dL0 + cnt[1] * dL1 + cnt[2] * dL2);
            }
            left = jout;
          }
        }
      }
    }
  }

  if (kSplit) {
    // both halves computed the same setups: the same warp maximum Tw; half 1
    // starts at step J = ceil(Tw / 2) from the walk's exact state there
    const int J = (__reduce_max_sync(0xffffffffu, left) + 1) / 2;
    if (half == 0) {
      left = min(left, J);
    } else if (left > J) {
      const float eb[3] = {(float)(sp.S[0] + (f0 >= 0.f ? 1 : 0)),
                           (float)(sp.S[1] + (f1 >= 0.f ? 1 : 0)),
                           (float)(sp.S[2] + (f2 >= 0.f ? 1 : 0))};
      const float fb[3] = {f0, f1, f2}, s3[3] = {s0, s1, s2}, inv[3] = {i0, i1, i2};
      const int jm[3] = {jm0, jm1, jm2};
      int c[3];
      const int nf = seek_prefix(eb, fb, s3, inv, jm, J, c);
      e0 = __fadd_rn(eb[0], f0 * (float)c[0]);
      e1 = __fadd_rn(eb[1], f1 * (float)c[1]);
      e2 = __fadd_rn(eb[2], f2 * (float)c[2]);
      k0 = jm0 > 0 ? __fmul_rn(__fsub_rn(e0, s0), i0) : kInf;
      k1 = jm1 > 0 ? __fmul_rn(__fsub_rn(e1, s1), i1) : kInf;
      k2 = jm2 > 0 ? __fmul_rn(__fsub_rn(e2, s2), i2) : kInf;
      L += (uint32_t)(c[0] * dL0 + c[1] * dL1 + c[2] * dL2);
      for (int t = 0; t < nf; ++t)  // the last events of the prefix, exact step rule
        dda_step(k0, k1, k2, e0, e1, e2, f0, f1, f2, i0, i1, i2, s0, s1, s2, dL0, dL1, dL2, L);
      left -= J;
    } else {
      left = 0;
    }
  }
  // tile occupancy counts, one atomic per group of lanes in the same tile
  {
    const unsigned peers = __match_any_sync(0xffffffffu, newtile);
    if (newtile != 0xffffffffu && lane == __ffs(peers) - 1)
      atomicAdd(tc.tile + newtile, (uint32_t)__popc(peers));
  }
  const unsigned after_lanes = 0xfffffffeu << lane;  // lanes above this one
  if (kSlab) {
    walk_loop_range<kStream, kNeg>(miss, L, jin, left, lane, after_lanes, [&] {
      dda_step(k0, k1, k2, e0, e1, e2, f0, f1, f2, i0, i1, i2, s0, s1, s2, dL0, dL1, dL2, L);
    });
    return;
  }
  walk_loop<kStream, kNeg>(miss, L, left, lane, after_lanes, [&] {
    dda_step(k0, k1, k2, e0, e1, e2, f0, f1, f2, i0, i1, i2, s0, s1, s2, dL0, dL1, dL2, L);
  });
}

// Block size: 64 threads (two adjacent rings) when the frame is about one
// wave of warps -- many small blocks spread long and short rings over the
// SMs -- and 128 (four adjacent rings) for multi-wave frames, where the
// locality of adjacent rings wins (c4 / c5: -7% / -4%; c2: +6% with 128).
// The bound (kBS, 1) lets ptxas spend 68 registers (59 under a 256-thread
// bound), which measured 8% faster on c5 and equal on c2; higher occupancy
// (40 / 48 warps per SM at 48 / 40 registers) measured slower on every config.
// kNeg: misses count down from -1 in the slot's LUT (the integrate path, see
// k_finalize_lut); else up from 0 in a plain miss grid (the multi-GPU partial
// grids that are reduce-scattered).
#ifndef GVOM_RAY_MINB64
#define GVOM_RAY_MINB64 1  // min resident 64-thread ray-cast blocks per SM (A/B builds)
#endif
template <bool kStream, int kBS, bool kNeg>
__global__ void __launch_bounds__(kBS, kBS == 64 ? GVOM_RAY_MINB64 : 1) k_raycast(const __grid_constant__ RayBatch rb,
                                                 const Dims d, uint32_t* __restrict__ miss,
                                                 uint32_t* __restrict__ bits,
                                                 const TileCounts tc, bool last_sensor) {
  ray_warp<kStream, kNeg>(rb, d, miss, bits, tc, (int64_t)blockIdx.x * blockDim.x + threadIdx.x);
  if (last_sensor && bits) scan_tiles_if_last(tc, d);
}

// Two warps per 32 rays (kSplit, GVOM_RAY_SPLIT=1): warp pair (2w, 2w+1) of the
// block walks the first / second half of ray warp w's steps.
template <bool kStream, int kBS, bool kNeg>
__global__ void __launch_bounds__(kBS, 1) k_raycast_split(const __grid_constant__ RayBatch rb,
                                                       const Dims d, uint32_t* __restrict__ miss,
                                                       uint32_t* __restrict__ bits,
                                                       const TileCounts tc, bool last_sensor) {
  const int w = threadIdx.x >> 5;
  const int64_t wtile = ((int64_t)blockIdx.x * (kBS / 32) + w) >> 1;
  ray_warp<kStream, kNeg, false, true>(rb, d, miss, bits, tc, wtile * 32 + (threadIdx.x & 31),
                                       SlabRange{0, 0}, w & 1);
  if (last_sensor && bits) scan_tiles_if_last(tc, d);
}

// Ray cast of the ray-segment slab partition: every ray of the frame, traced
// only inside rows [sr.y0, sr.y1) (SURVEY 8(e) reworked).
template <bool kStream, int kBS>
__global__ void __launch_bounds__(kBS, 1) k_raycast_slab(const __grid_constant__ RayBatch rb,
                                                      const Dims d, uint32_t* __restrict__ miss,
                                                      uint32_t* __restrict__ bits,
                                                      const TileCounts tc, bool last_sensor,
                                                      const SlabRange sr) {
  ray_warp<kStream, true, true>(rb, d, miss, bits, tc,
                                (int64_t)blockIdx.x * blockDim.x + threadIdx.x, sr);
  if (last_sensor && bits) scan_tiles_if_last(tc, d);
}

// Single-pass rank of the occupied voxels (decoupled look-back scan over the
// occupancy bitmask): absolute exclusive popcount prefix per 32-voxel word, so
// rank(L) = wprefix[L>>5] + popc(bits[L>>5] & ((1<<(L&31))-1)) is the voxel's
// index in L order (reading A2, deterministic).  Tiles are taken in launch
// order from a ticket counter; status words carry an epoch so nothing needs
// resetting between calls.
constexpr uint64_t kFlagIncl = 1ull << 32;

__device__ __forceinline__ uint64_t ld_acquire(const uint64_t* p) {
  return cuda::atomic_ref<const uint64_t, cuda::thread_scope_device>(*p).load(
      cuda::memory_order_acquire);
}
__device__ __forceinline__ void st_release(uint64_t* p, uint64_t v) {
  cuda::atomic_ref<uint64_t, cuda::thread_scope_device>(*p).store(v, cuda::memory_order_release);
}

__global__ void __launch_bounds__(kRankThreads) k_rank(const uint32_t* __restrict__ bits,
                                                       int64_t W, uint32_t* __restrict__ wprefix,
                                                       uint64_t* __restrict__ status,
                                                       unsigned long long* __restrict__ ticket,
                                                       uint64_t base, uint32_t epoch,
                                                       int64_t nblk,
                                                       uint32_t* __restrict__ total_out) {
  __shared__ uint32_t wsum[kRankThreads / 32];
  __shared__ uint32_t sprefix;
  __shared__ int64_t sbid;
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  if (t == 0) sbid = (int64_t)(atomicAdd(ticket, 1ull) - base);
  __syncthreads();
  const int64_t bid = sbid;
  const int64_t w0 = bid * kRankWordsPerBlock + t * 4;
  uint32_t w4[4];
  if (w0 + 3 < W) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(bits + w0));
    w4[0] = v.x;
    w4[1] = v.y;
    w4[2] = v.z;
    w4[3] = v.w;
  } else {
    for (int i = 0; i < 4; ++i) w4[i] = (w0 + i < W) ? bits[w0 + i] : 0u;
  }
  const uint32_t c0 = __popc(w4[0]), c1 = __popc(w4[1]), c2 = __popc(w4[2]), c3 = __popc(w4[3]);
  const uint32_t tsum = c0 + c1 + c2 + c3;
  const uint32_t inc = warp_incl_scan(tsum, lane);
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const uint32_t v = lane < kRankThreads / 32 ? wsum[lane] : 0u;
    const uint32_t i = warp_incl_scan(v, lane);
    if (lane < kRankThreads / 32) wsum[lane] = i - v;  // exclusive per warp
    const uint32_t total = __shfl_sync(0xffffffffu, i, kRankThreads / 32 - 1);
    const uint64_t ep = (uint64_t)epoch << 33;
    if (bid == 0) {
      if (lane == 0) {
        st_release(status, ep | kFlagIncl | total);
        sprefix = 0;
      }
    } else {
      if (lane == 0) st_release(status + bid, ep | total);
      // look back over predecessors, 32 at a time
      uint32_t prefix = 0;
      int64_t jb = bid - 1;
      for (;;) {
        const int64_t j = jb - lane;
        uint64_t sv = j >= 0 ? ld_acquire(status + j) : (ep | kFlagIncl);
        while (__any_sync(0xffffffffu, (sv >> 33) != epoch)) {
          if ((sv >> 33) != epoch) sv = ld_acquire(status + j);
        }
        const unsigned incl = __ballot_sync(0xffffffffu, (sv & kFlagIncl) != 0);
        const int stop = incl ? __ffs(incl) - 1 : 31;  // nearest inclusive predecessor
        uint32_t val = lane <= stop ? (uint32_t)sv : 0u;
        val = __reduce_add_sync(0xffffffffu, val);
        prefix += val;
        if (incl) break;
        jb -= 32;
      }
      if (lane == 0) {
        st_release(status + bid, ep | kFlagIncl | (prefix + total));
        sprefix = prefix;
      }
    }
    if (lane == 0 && bid == nblk - 1) *total_out = (bid == 0 ? 0u : sprefix) + total;
  }
  __syncthreads();
  const uint32_t p0 = sprefix + wsum[wid] + inc - tsum;
  if (w0 + 3 < W) {
    *reinterpret_cast<uint4*>(wprefix + w0) = make_uint4(p0, p0 + c0, p0 + c0 + c1,
                                                         p0 + c0 + c1 + c2);
  } else {
    const uint32_t pp[4] = {p0, p0 + c0, p0 + c0 + c1, p0 + c0 + c1 + c2};
    for (int i = 0; i < 4; ++i)
      if (w0 + i < W) wprefix[w0 + i] = pp[i];
  }
}

// Zero three regions in one launch (the slot's LUT-as-miss-grid, its
// occupancy bitmask, and the tile counters).  The miss grid is written
// evict-first, except (keep_a) for large grids that still fit in L2 (32-96
// MiB): there write-back zeros leave the grid in L2 for the ray cast's REDs
// (c4, 64 MiB: step 256 -> 248 us); the small c2 grid measured 1.5% slower
// with write-back.
__global__ void __launch_bounds__(256) k_zero3(uint4* __restrict__ a, int64_t na,
                                               uint4* __restrict__ b, int64_t nb,
                                               uint4* __restrict__ c, int64_t nc, bool keep_a) {
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na + nb + nc; i += stride) {
    if (i < na) {
      if (keep_a)
        a[i] = z;
      else
        __stcs(a + i, z);
    }
    else if (i < na + nb)
      __stcs(b + (i - na), z);
    else
      __stcs(c + (i - na - nb), z);
  }
}

// Rank + O6 encode in one launch (O6: buf[L] holds the miss count and
// becomes the rank if occupied, else -1 - min(N_m, 2^30); occupied rows get
// {0, misses, 0xFFFFFFFF, 0, 0, 0} for the endpoint pass).  Block b owns tile
// b (256 bitmask words = 8192 voxels): its rank offset is the exclusive
// prefix of the tile counts kept by the ray cast and scanned by its last
// block, so no block waits on another.  Then: per-word prefix (block scan),
// wprefix store, and the in-place LUT encode / data-row init of its 8192
// voxels with 16-byte accesses.
// kPeers (NEXT-2, fused collective): the miss count of voxel L is the sum of
// the P ranks' partial grids peers.g[p][L], read over peer memory as the tile
// is encoded -- the reduce-scatter of the grids fused into the finalize.
template <bool kPeers>
__device__ __forceinline__ uint4 miss4(const int32_t* __restrict__ buf, const PeerGrids& peers,
                                       int64_t L) {
  if (!kPeers) return __ldcs(reinterpret_cast<const uint4*>(buf + L));
  uint4 s = make_uint4(0u, 0u, 0u, 0u);
  for (int p = 0; p < peers.P; ++p) {
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(peers.g[p] + L));
    s.x += v.x;
    s.y += v.y;
    s.z += v.z;
    s.w += v.w;
  }
  return s;
}
template <bool kPeers>
__device__ __forceinline__ uint32_t miss1(const int32_t* __restrict__ buf, const PeerGrids& peers,
                                          int64_t L) {
  if (!kPeers) return (uint32_t)buf[L];
  uint32_t s = 0;
  for (int p = 0; p < peers.P; ++p) s += __ldcs(peers.g[p] + L);
  return s;
}

template <bool kPeers>
__global__ void __launch_bounds__(kTileWords) k_finalize_tiles(
    int32_t* __restrict__ buf, const uint32_t* __restrict__ bits, uint32_t* __restrict__ wprefix,
    gvom_voxel* __restrict__ data, const TileCounts tc, const Dims d, int64_t t_begin,
    uint32_t base, const __grid_constant__ PeerGrids peers) {
  __shared__ uint32_t sbits[kTileWords], spre[kTileWords], wsum[kTileWords / 32];
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t b = t_begin + blockIdx.x;
  const uint32_t off = base + __ldg(tc.offset + b);  // rank offset of this tile
  // per-word exclusive prefix within the tile
  const int64_t w = b * kTileWords + t;
  const uint32_t bw = w < d.W ? __ldg(bits + w) : 0u;
  const uint32_t c = __popc(bw);
  const uint32_t inc = warp_incl_scan(c, lane);
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const uint32_t v = lane < kTileWords / 32 ? wsum[lane] : 0u;
    const uint32_t e = warp_incl_scan(v, lane) - v;
    if (lane < kTileWords / 32) wsum[lane] = e;
  }
  __syncthreads();
  const uint32_t pre = off + wsum[wid] + inc - c;
  sbits[t] = bw;
  spre[t] = pre;
  if (w < d.W) wprefix[w] = pre;
  if (blockIdx.x == gridDim.x - 1 && t == kTileWords - 1) *tc.total = pre + c;  // k of the frame
  __syncthreads();
  // voxels of the tile: 8 x 16-byte chunks per thread, all loads in flight
  // before any store (the tile is whole unless it is the grid's last)
  const int64_t vbase = b << kTileShift;
  constexpr int kIt = (1 << kTileShift) / (kTileWords * 4);  // 8
  if (vbase + (1 << kTileShift) <= d.V) {
    uint4 mv[kIt];
#pragma unroll
    for (int it = 0; it < kIt; ++it)
      mv[it] = miss4<kPeers>(buf, peers, vbase + t * 4 + it * kTileWords * 4);
#pragma unroll
    for (int it = 0; it < kIt; ++it) {
      const int i = t * 4 + it * kTileWords * 4;
      const uint32_t ww = sbits[i >> 5], pp = spre[i >> 5];
      const uint32_t m[4] = {mv[it].x, mv[it].y, mv[it].z, mv[it].w};
      int32_t o[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int bit = (i + j) & 31;
        if ((ww >> bit) & 1u) {
          const uint32_t rank = pp + __popc(ww & ((1u << bit) - 1u));
          o[j] = (int32_t)rank;
          uint4* row = reinterpret_cast<uint4*>(data + rank);
          row[0] = make_uint4(0u, m[j], 0xffffffffu, 0u);
          row[1] = make_uint4(0u, 0u, 0u, 0u);
        } else {
          o[j] = -1 - (int32_t)(m[j] < kMissSat ? m[j] : kMissSat);
        }
      }
      *reinterpret_cast<int4*>(buf + vbase + i) = make_int4(o[0], o[1], o[2], o[3]);
    }
    return;
  }
  for (int i = t * 4; i < (1 << kTileShift); i += kTileWords * 4) {
    const int64_t L = vbase + i;
    if (L >= d.V) break;
    const uint32_t ww = sbits[i >> 5], pp = spre[i >> 5];
    uint32_t m[4];
    for (int j = 0; j < 4; ++j) m[j] = (L + j < d.V) ? miss1<kPeers>(buf, peers, L + j) : 0u;
    for (int j = 0; j < 4; ++j) {
      if (L + j >= d.V) break;
      const int bit = (i + j) & 31;
      if ((ww >> bit) & 1u) {
        const uint32_t rank = pp + __popc(ww & ((1u << bit) - 1u));
        buf[L + j] = (int32_t)rank;
        uint4* row = reinterpret_cast<uint4*>(data + rank);
        row[0] = make_uint4(0u, m[j], 0xffffffffu, 0u);
        row[1] = make_uint4(0u, 0u, 0u, 0u);
      } else {
        buf[L + j] = -1 - (int32_t)(m[j] < kMissSat ? m[j] : kMissSat);
      }
    }
  }
}

// O4 per return: hits, min_dz, m1 = sum dz, m2 = sum dz^2 into the data row.
// Returns of azimuth-adjacent lanes often share a voxel (ground near the
// sensor): runs of equal voxels are reduced with a segmented shuffle
// reduction and the run head issues the four atomics.  Only returns in the
// rows of `sr` are binned (the whole map, or a rank's slab).
__device__ __forceinline__ void endpoint_warp(const RayBatch& rb, const Dims& d, int64_t gtid,
                                              const int32_t* __restrict__ lut,
                                              gvom_voxel* __restrict__ data,
                                              const SlabRange sr) {
  // the batch's sensors interleaved by 32-column tile, as in k_raycast
  const int64_t gt = gtid / rb.tile_threads;
  const int sidx = (int)(gt % rb.S);
  const int64_t tid = (gt / rb.S) * rb.tile_threads + (gtid - gt * rb.tile_threads);
  const int64_t n = rb.n[sidx];
  const float4* __restrict__ pts = rb.pts[sidx];
  const SensorParams& sp = rb.sp[sidx];
  const int64_t p = point_index(tid, rb.rings);
  const int lane = threadIdx.x & 31;
  bool valid = false;
  uint32_t LE = 0xffffffffu, dz = 0u;
  if (p < n) {
    const float4 q = __ldg(pts + p);
    float g0, g1, g2;
    if (transform_point(sp, q, g0, g1, g2)) {
      const int e0 = (int)floorf(g0), e1 = (int)floorf(g1), e2 = (int)floorf(g2);
      if ((unsigned)e0 < (unsigned)d.nx && e1 >= sr.y0 && e1 < sr.y1 &&
          (unsigned)e2 < (unsigned)d.nz) {
        valid = true;
        LE = (uint32_t)(e2 + d.nz * e0 + d.nz * d.nx * e1);
        // qz = floor(f32(g_z * 65536)) is exact (power-of-two scale)
        const int64_t qz = (int64_t)floorf(__fmul_rn(g2, 65536.0f));
        dz = (uint32_t)(qz - 65536ll * e2);
      }
    }
  }
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  if (act == 0u) return;  // warp-uniform
  const uint32_t prev = __shfl_up_sync(0xffffffffu, LE, 1);
  const bool head = valid && (lane == 0 || prev != LE);
  const unsigned heads = __ballot_sync(0xffffffffu, head);
  const int end = __clz(__brev((heads | ~act) & (0xfffffffeu << lane))) - 1;  // run's last lane
  uint32_t cnt = valid ? 1u : 0u, s1 = dz, mn = valid ? dz : 0xffffffffu;
  uint64_t s2 = (uint64_t)dz * dz;
  // every valid lane its own run (far returns): nothing to reduce
  if (heads != act)
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t c_o = __shfl_down_sync(0xffffffffu, cnt, o);
    const uint32_t s1_o = __shfl_down_sync(0xffffffffu, s1, o);
    const uint64_t s2_o = __shfl_down_sync(0xffffffffu, s2, o);
    const uint32_t mn_o = __shfl_down_sync(0xffffffffu, mn, o);
    if (lane + o <= end) {
      cnt += c_o;
      s1 += s1_o;
      s2 += s2_o;
      mn = min(mn, mn_o);
    }
  }
  if (head) {
    const int32_t rank = __ldg(lut + LE);
    gvom_voxel* row = data + rank;
    atomicAdd(&row->hits, cnt);
    atomicMin(&row->min_dz, mn);
    atomicAdd(reinterpret_cast<unsigned long long*>(&row->m1), (unsigned long long)s1);
    atomicAdd(reinterpret_cast<unsigned long long*>(&row->m2), (unsigned long long)s2);
  }
}

__global__ void __launch_bounds__(256) k_endpoint(const __grid_constant__ RayBatch rb,
                                                  const Dims d, const int32_t* __restrict__ lut,
                                                  gvom_voxel* __restrict__ data,
                                                  const SlabRange sr) {
  endpoint_warp(rb, d, (int64_t)blockIdx.x * blockDim.x + threadIdx.x, lut, data, sr);
}

// Integrate pass 0: the slot's LUT over tiles [t0, t1) set to -1 ("empty, no
// misses", O6) and its occupancy bits cleared.  The ray cast then counts each
// pass-through DOWN from -1 in place (kNeg), so an empty voxel's LUT entry is
// already its final O6 code -1 - N_m (N_m <= points per frame <= 2^30: the
// 2^30 saturation never applies, gvom_create checks the capacity), and the
// finalize touches only occupied voxels.  Write-back stores for a LUT that
// fits in L2 (the ray cast's reductions then hit L2), evict-first beyond.
template <bool kKeep>
__global__ void __launch_bounds__(256) k_reset_slot(int32_t* __restrict__ lut, int64_t l0,
                                                    int64_t l1, uint32_t* __restrict__ bits,
                                                    int64_t w0, int64_t w1) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // l0, w0 are tile starts: 16-byte aligned; tails (l1, w1 not multiples of 4) scalar
  const int64_t n4 = (l1 - l0) >> 2, m4 = (w1 - w0) >> 2;
  const int4 ones = make_int4(-1, -1, -1, -1);
  int4* l4 = reinterpret_cast<int4*>(lut + l0);
  int64_t i = i0;
#if GVOM_RESET_V8
  {  // 32-byte stores (STG.256; l0 is a tile start: 32 KB aligned), four in flight
    const int64_t n8 = n4 >> 1;
    char* l8 = reinterpret_cast<char*>(lut + l0);
    int64_t k = i0;
    for (; k + 3 * stride < n8; k += 4 * stride) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        char* a = l8 + 32 * (k + u * stride);
        if (kKeep)
          asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(a), "r"(-1)
                       : "memory");
        else
          asm volatile("st.global.cs.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(a), "r"(-1)
                       : "memory");
      }
    }
    for (; k < n8; k += stride) {
      char* a = l8 + 32 * k;
      if (kKeep)
        asm volatile("st.global.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(a), "r"(-1)
                     : "memory");
      else
        asm volatile("st.global.cs.v8.b32 [%0], {%1,%1,%1,%1,%1,%1,%1,%1};" ::"l"(a), "r"(-1)
                     : "memory");
    }
    i = 2 * n8 + i0;  // the odd 16-byte chunk, if any, below
  }
#endif
  for (; i + 3 * stride < n4; i += 4 * stride) {  // four 16-byte stores in flight
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if (kKeep)
        l4[i + u * stride] = ones;
      else
        __stcs(l4 + i + u * stride, ones);
    }
  }
  for (; i < n4; i += stride) {
    if (kKeep)
      l4[i] = ones;
    else
      __stcs(l4 + i, ones);
  }
  uint4* b4 = reinterpret_cast<uint4*>(bits + w0);
  for (int64_t j = i0; j < m4; j += stride) __stcs(b4 + j, make_uint4(0u, 0u, 0u, 0u));
  if (i0 < 4) {
    if (l0 + 4 * n4 + i0 < l1) lut[l0 + 4 * n4 + i0] = -1;
    if (w0 + 4 * m4 + i0 < w1) bits[w0 + 4 * m4 + i0] = 0u;
  }
}

// Integrate pass 1 (O6) over tiles [t0, t0 + gridDim.x): block b owns tile b
// (256 bitmask words = 8192 voxels); its rank offset is the exclusive prefix
// of the tile counts the ray cast kept and scanned, so no block waits on
// another.  Per-word prefix (block scan) -> wprefix; each thread lists its
// word's occupied voxels in shared memory at their rank within the tile, then
// the block walks that list -- one occupied voxel per thread, loads
// independent: the LUT entry holds -1 - misses (counted down by the ray
// cast), it becomes the voxel's rank and its data row {0, misses, 0xFFFFFFFF,
// 0, 0, 0} is initialised for the endpoint pass.  Empty voxels' entries are
// final already.
// (Binning the returns in the same launch, endpoint blocks waiting on per-tile
// flags, measured slower: c2 integrate 83-86 vs 75-78 us; again in round 2
// with blocks ordered by a ticket so tile blocks start first: c2 step 115 vs
// 108 us, c3 137 vs 132 us -- the finalize launch's tail then holds the
// endpoint blocks' waits.)
__global__ void __launch_bounds__(kTileWords) k_finalize_lut(
    int32_t* __restrict__ lut, const uint32_t* __restrict__ bits, uint32_t* __restrict__ wprefix,
    gvom_voxel* __restrict__ data, const TileCounts tc, const Dims d, int64_t t0) {
  __shared__ uint32_t wsum[kTileWords / 32];
  __shared__ uint16_t slist[1 << kTileShift];  // occupied voxels of the tile, rank order
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t bl = blockIdx.x;
  const int64_t b = t0 + bl;
  const uint32_t off = __ldg(tc.offset + b);  // rank offset of this tile
  const int64_t w = b * kTileWords + t;
  const uint32_t bw = w < d.W ? __ldg(bits + w) : 0u;
  const uint32_t c = __popc(bw);
  const uint32_t inc = warp_incl_scan(c, lane);
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const uint32_t v = lane < kTileWords / 32 ? wsum[lane] : 0u;
    const uint32_t i = warp_incl_scan(v, lane);
    if (lane < kTileWords / 32) wsum[lane] = i - v;
  }
  __syncthreads();
  const uint32_t rel = wsum[wid] + inc - c;  // rank of the word's first voxel in the tile
  const uint32_t pre = off + rel;
  if (w < d.W) wprefix[w] = pre;
  if (t == 0) tc.tile[b] = 0u;  // consumed by the ray cast's scan: zero for the next frame
  uint32_t m = bw, j = rel;
  while (m) {
    slist[j++] = (uint16_t)(t * 32 + __ffs(m) - 1);
    m &= m - 1u;
  }
  __shared__ uint32_t stotal;
  if (t == kTileWords - 1) {
    stotal = rel + c;
    if (bl == gridDim.x - 1) *tc.total = pre + c;  // k of the frame
  }
  __syncthreads();
  const uint32_t n = stotal;
  const int64_t vbase = b << kTileShift;
  // eight list entries per thread at a time: all their loads in flight before
  // any store (a dense tile -- ground near the sensor -- holds thousands)
  constexpr int kU = 8;
  for (uint32_t i0 = t; i0 < n; i0 += kU * kTileWords) {
    int32_t v[kU];
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t i = i0 + u * kTileWords;
      v[u] = i < n ? __ldcg(lut + vbase + slist[i]) : 0;
    }
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const uint32_t i = i0 + u * kTileWords;
      if (i >= n) break;
      const uint32_t rank = off + i;
      lut[vbase + slist[i]] = (int32_t)rank;
      uint4* row = reinterpret_cast<uint4*>(data + rank);
      row[0] = make_uint4(0u, (uint32_t)(-1 - v[u]), 0xffffffffu, 0u);
      row[1] = make_uint4(0u, 0u, 0u, 0u);
    }
  }
}

inline int64_t point_threads(int64_t n, int32_t rings) {
  if (rings <= 1) return n;
  const int64_t cols = (n + rings - 1) / rings;
  const int64_t tiles = (cols + 31) / 32;
  return tiles * 32 * rings;
}

}  // namespace

#ifndef GVOM_RAY_NARROW_BS
#define GVOM_RAY_NARROW_BS 64
#endif
constexpr int kRayNarrowBS = GVOM_RAY_NARROW_BS;  // block size of one-wave frames (A/B switch)

template <bool kNeg>
static void launch_raycast_t(bool stream, bool wide, unsigned blocks, const RayBatch& rb,
                             const Dims& d, uint32_t* miss, uint32_t* bits, const TileCounts& tc,
                             bool last, cudaStream_t st) {
  if (!stream && !wide)
    k_raycast<false, kRayNarrowBS, kNeg><<<blocks, kRayNarrowBS, 0, st>>>(rb, d, miss, bits, tc,
                                                                          last);
  else if (!stream)
    k_raycast<false, 128, kNeg><<<blocks, 128, 0, st>>>(rb, d, miss, bits, tc, last);
  else if (!wide)
    k_raycast<true, kRayNarrowBS, kNeg><<<blocks, kRayNarrowBS, 0, st>>>(rb, d, miss, bits, tc,
                                                                         last);
  else
    k_raycast<true, 128, kNeg><<<blocks, 128, 0, st>>>(rb, d, miss, bits, tc, last);
}

cudaError_t launch_raycast(const RayBatch& rb, const Dims& d, uint32_t* miss_grid,
                           uint32_t* bits, const TileCounts& tc, bool last_launch,
                           cudaStream_t st, const SlabRange* slab, bool lut_direct) {
  int64_t tiles = 0;  // per sensor, the batch's maximum
  for (int s = 0; s < rb.S; ++s) {
    const int64_t t = (point_threads(rb.n[s], rb.rings) + rb.tile_threads - 1) / rb.tile_threads;
    tiles = t > tiles ? t : tiles;
  }
  const int64_t threads = tiles * rb.S * rb.tile_threads;
  if (threads == 0) return cudaSuccess;
  // block size by frame size (see k_raycast): more than one wave of warps
  // (SMs x 30 resident warps) -> 128 threads, else 64
  // (round 2: above ONE wave -- c3, 1.85 waves, ray cast 68.8 vs 70.4 us with
  // the 128-thread split kernel; GVOM_RAY_WIDE_WAVES: the threshold, A/B)
  static int wide_waves = -1;
  if (wide_waves < 0) {
    const char* e = getenv("GVOM_RAY_WIDE_WAVES");
    wide_waves = e ? atoi(e) : 1;
  }
  const bool wide = threads / 32 > (int64_t)wide_waves * d.sms * 30;
  const int bs = wide ? 128 : kRayNarrowBS;
  const unsigned blocks = (unsigned)((threads + bs - 1) / bs);
  // schedule by where the REDs land (see aggregate_red_*): the resident one
  // also needs byte offsets < 2^32
  const int64_t miss_bytes = (int64_t)d.nx * d.ny * d.nz * 4;
  const int64_t resident_max = kRayStreamBytes > 0 ? kRayStreamBytes : d.l2_bytes / 2;
  const bool stream = !(miss_bytes <= resident_max && miss_bytes < (int64_t(1) << 32));
  if (slab && (slab->y0 > 0 || slab->y1 < d.ny)) {  // ray-segment slab partition (LUT-direct)
    if (!stream && !wide)
      k_raycast_slab<false, kRayNarrowBS><<<blocks, kRayNarrowBS, 0, st>>>(
          rb, d, miss_grid, bits, tc, last_launch, *slab);
    else if (!stream)
      k_raycast_slab<false, 128><<<blocks, 128, 0, st>>>(rb, d, miss_grid, bits, tc, last_launch,
                                                         *slab);
    else if (!wide)
      k_raycast_slab<true, kRayNarrowBS><<<blocks, kRayNarrowBS, 0, st>>>(
          rb, d, miss_grid, bits, tc, last_launch, *slab);
    else
      k_raycast_slab<true, 128><<<blocks, 128, 0, st>>>(rb, d, miss_grid, bits, tc, last_launch,
                                                        *slab);
    return cudaGetLastError();
  }
  // two warps per 32 rays for the wide frames (c3 -2 %, c4 -3 %, c5 -4 %;
  // one-wave frames lose: c2 +7 %); GVOM_RAY_SPLIT=0 / 1 forces it
  static int split_env = -2;
  if (split_env == -2) {
    const char* e = getenv("GVOM_RAY_SPLIT");
    split_env = e ? (atoi(e) ? 1 : 0) : -1;
  }
  const bool split = split_env >= 0 ? split_env == 1 : wide;
  if (split && lut_direct) {
    const unsigned b2 = (unsigned)((2 * threads + bs - 1) / bs);
    if (!stream && !wide)
      k_raycast_split<false, kRayNarrowBS, true><<<b2, kRayNarrowBS, 0, st>>>(
          rb, d, miss_grid, bits, tc, last_launch);
    else if (!stream)
      k_raycast_split<false, 128, true><<<b2, 128, 0, st>>>(rb, d, miss_grid, bits, tc,
                                                            last_launch);
    else if (!wide)
      k_raycast_split<true, kRayNarrowBS, true><<<b2, kRayNarrowBS, 0, st>>>(
          rb, d, miss_grid, bits, tc, last_launch);
    else
      k_raycast_split<true, 128, true><<<b2, 128, 0, st>>>(rb, d, miss_grid, bits, tc,
                                                           last_launch);
    return cudaGetLastError();
  }
  if (lut_direct)
    launch_raycast_t<true>(stream, wide, blocks, rb, d, miss_grid, bits, tc, last_launch, st);
  else
    launch_raycast_t<false>(stream, wide, blocks, rb, d, miss_grid, bits, tc, last_launch, st);
  return cudaGetLastError();
}

cudaError_t launch_rank(const uint32_t* bits, const Dims& d, uint32_t* wprefix, uint64_t* status,
                        unsigned long long* ticket, uint64_t base, uint32_t epoch,
                        uint32_t* total, cudaStream_t st) {
  const int64_t nblk = rank_blocks(d);
  k_rank<<<(unsigned)nblk, kRankThreads, 0, st>>>(bits, d.W, wprefix, status, ticket, base, epoch,
                                                   nblk, total);
  return cudaGetLastError();
}

// miss grids zeroed write-back: (L2/4, 3 L2/4] (B200, 126 MB: ~32-95 MB)
cudaError_t launch_zero3(void* a, size_t abytes, void* b, size_t bbytes, void* c, size_t cbytes,
                         const Dims& d, cudaStream_t st) {
  const int64_t n = (int64_t)(abytes / 16 + bbytes / 16 + cbytes / 16);
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)d.sms * 8) blocks = (int64_t)d.sms * 8;
  if (blocks < 1) blocks = 1;
  const bool keep_a = (int64_t)abytes > d.l2_bytes / 4 && (int64_t)abytes <= 3 * d.l2_bytes / 4;
  k_zero3<<<(unsigned)blocks, 256, 0, st>>>((uint4*)a, (int64_t)(abytes / 16), (uint4*)b,
                                            (int64_t)(bbytes / 16), (uint4*)c,
                                            (int64_t)(cbytes / 16), keep_a);
  return cudaGetLastError();
}

cudaError_t launch_finalize_tiles(int32_t* lut_inplace, const uint32_t* bits, uint32_t* wprefix,
                                  gvom_voxel* data, const TileCounts& tc, const Dims& d,
                                  cudaStream_t st, int64_t t_begin, int64_t t_end, uint32_t base,
                                  const PeerGrids* peers) {
  if (t_end < 0) t_end = n_tiles(d);
  if (t_end <= t_begin) return cudaSuccess;
  const unsigned grid = (unsigned)(t_end - t_begin);
  if (peers && peers->P > 0) {
    k_finalize_tiles<true><<<grid, kTileWords, 0, st>>>(lut_inplace, bits, wprefix, data, tc, d,
                                                       t_begin, base, *peers);
  } else {
    PeerGrids none{};
    k_finalize_tiles<false><<<grid, kTileWords, 0, st>>>(lut_inplace, bits, wprefix, data, tc, d,
                                                        t_begin, base, none);
  }
  return cudaGetLastError();
}

cudaError_t launch_reset_slot(int32_t* lut, uint32_t* bits, const Dims& d, int64_t t0,
                              int64_t t1, cudaStream_t st) {
  const int64_t l0 = t0 << kTileShift, l1 = min(d.V, t1 << kTileShift);
  const int64_t w0 = t0 * kTileWords, w1 = min(d.W, t1 * kTileWords);
  if (l1 <= l0) return cudaSuccess;
  const int64_t n = (l1 - l0) / 4 + (w1 - w0) / 4;
  int64_t blocks = (n + 255) / 256;
  if (blocks > (int64_t)d.sms * 8) blocks = (int64_t)d.sms * 8;
  if (blocks < 1) blocks = 1;
  static int use_memset = -1;  // GVOM_RESET_MEMSET=1: two driver memsets (A/B)
  if (use_memset < 0) {
    const char* e = getenv("GVOM_RESET_MEMSET");
    use_memset = e && atoi(e) ? 1 : 0;
  }
  if (use_memset) {
    cudaError_t e = cudaMemsetAsync(lut + l0, 0xff, 4 * (size_t)(l1 - l0), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(bits + w0, 0, 4 * (size_t)(w1 - w0), st);
    return e;
  }
  const bool keep = 4 * (l1 - l0) <= 3 * d.l2_bytes / 4;  // the REDs then hit L2
  if (keep)
    k_reset_slot<true><<<(unsigned)blocks, 256, 0, st>>>(lut, l0, l1, bits, w0, w1);
  else
    k_reset_slot<false><<<(unsigned)blocks, 256, 0, st>>>(lut, l0, l1, bits, w0, w1);
  return cudaGetLastError();
}

cudaError_t launch_finalize_lut(int32_t* lut, const uint32_t* bits, uint32_t* wprefix,
                                gvom_voxel* data, const TileCounts& tc, const Dims& d, int64_t t0,
                                int64_t t1, cudaStream_t st) {
  if (t1 <= t0) return cudaSuccess;
  k_finalize_lut<<<(unsigned)(t1 - t0), kTileWords, 0, st>>>(lut, bits, wprefix, data, tc, d, t0);
  return cudaGetLastError();
}

cudaError_t launch_endpoint(const RayBatch& rb, const Dims& d, const int32_t* lut,
                            gvom_voxel* data, cudaStream_t st, const SlabRange& slab) {
  int64_t tiles = 0;  // per sensor, the batch's maximum
  for (int s = 0; s < rb.S; ++s) {
    const int64_t t = (point_threads(rb.n[s], rb.rings) + rb.tile_threads - 1) / rb.tile_threads;
    tiles = t > tiles ? t : tiles;
  }
  const int64_t threads = tiles * rb.S * rb.tile_threads;
  if (threads == 0) return cudaSuccess;
  k_endpoint<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(rb, d, lut, data, slab);
  return cudaGetLastError();
}

}  // namespace gvom
