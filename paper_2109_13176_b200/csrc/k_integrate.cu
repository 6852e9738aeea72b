// k_integrate.cu -- pointcloud processing (section III.C) on sm_100a.
//
//   raycast  : transform + endpoint occupancy bit + float32 DDA pass-through counts
//   rank_*   : deterministic rank of occupied voxels in L order (LUT indices)
//   finalize : in-place LUT encode (rank | -1 - N_m) + data rows
//   endpoint : per-return hits, lowest return, fixed-point moments into data rows
//
// Numerics: every float op that decides an integer is written as an explicit
// IEEE round-to-nearest intrinsic (__fmul_rn/__fadd_rn/__fsub_rn/__frcp_rn) in
// the order of SURVEY.md 8(c) O3/O5, and the file is built with -fmad=false, so
// the voxel walk is bit-identical to the oracle's.  Integer accumulation only
// (u32/u64 atomics): results are independent of thread schedule.
#include <cuda/atomic>

#include "gvom_internal.cuh"

namespace gvom {

namespace {

constexpr float kGLim = 4194304.0f;  // |g_i| < 2^22 voxels (reading A5)

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

// O3: g_i = ((A_i0 x + A_i1 y) + A_i2 z) + b_i, f32 RN each, no contraction.
__device__ __forceinline__ bool transform_point(const SensorParams& sp, const float4 p,
                                                float& g0, float& g1, float& g2) {
  if (!isfinite(p.x) || !isfinite(p.y) || !isfinite(p.z)) return false;
  if (p.x == 0.0f && p.y == 0.0f && p.z == 0.0f) return false;
  float g[3];
#pragma unroll
  for (int i = 0; i < 3; ++i) {
    const float t0 = __fmul_rn(sp.A[3 * i + 0], p.x);
    const float t1 = __fmul_rn(sp.A[3 * i + 1], p.y);
    const float t2 = __fmul_rn(sp.A[3 * i + 2], p.z);
    g[i] = __fadd_rn(__fadd_rn(__fadd_rn(t0, t1), t2), sp.b[i]);
  }
  g0 = g[0];
  g1 = g[1];
  g2 = g[2];
  return fabsf(g0) < kGLim && fabsf(g1) < kGLim && fabsf(g2) < kGLim;
}

// Exact O5 walk of one ray, oracle control flow verbatim (slow path for the
// astronomically rare rays whose reciprocal 1/d_a is not finite, where the
// fast path's +inf-key gating would not be equivalent).
__device__ void walk_exact(const int S[3], const int E[3], const float g[3], const float s[3],
                           const Dims& d, uint32_t* __restrict__ miss) {
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
    atomicAdd(miss + (V[2] + d.nz * (V[0] + d.nx * V[1])), 1u);
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

// Per-axis DDA setup (O5).  The stateless key of the oracle,
//   key_a(V) = f32( f32( f32(V_a + [step_a>0]) - s_a ) * inv_a ),
// is evaluated from a float edge e_a = f32(V_a + [step_a>0]) that moves by
// exactly +-1 (integers < 2^24), so it is bit-identical.  Gating: an axis
// with no steps left carries key +inf; with every live key finite this picks
// exactly the oracle's argmin (strict <, ties to the lowest axis).
//   exit axis (the walk leaves the grid through it): c = in-grid steps left;
//   selecting it with c == 0 ends the walk.
//   other axes: c = rem; the key becomes +inf when c reaches 0.
__device__ __forceinline__ void axis_setup(int S, int E, float g, float s, int n, int stride,
                                           float& e, float& f, float& inv, float& key, int& c,
                                           int& dL, bool& x, int& rem, bool& finite) {
  const int st = (E > S) - (E < S);
  rem = abs(E - S);
  const int room = st > 0 ? (n - 1 - S) : S;  // in-grid steps available
  f = (float)st;
  // no steps on this axis: key (e - s) * inv = (S + 1 - s) * +inf = +inf
  e = (float)(S + (st >= 0 ? 1 : 0));
  inv = __int_as_float(0x7f800000);
  key = __int_as_float(0x7f800000);
  x = rem > room;
  c = x ? room : rem;
  if (rem > 0) {
    inv = __frcp_rn(__fsub_rn(g, s));
    key = __fmul_rn(__fsub_rn(e, s), inv);
    finite = finite && isfinite(inv);
  }
  dL = st * stride;
}

__global__ void __launch_bounds__(256) k_raycast(const float4* __restrict__ pts, int64_t n,
                                                 int32_t rings, const SensorParams sp,
                                                 const Dims d, uint32_t* __restrict__ miss,
                                                 uint32_t* __restrict__ bits) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p = point_index(tid, rings);
  const int lane = threadIdx.x & 31;
  const float s0 = sp.b[0], s1 = sp.b[1], s2 = sp.b[2];
  const float kInf = __int_as_float(0x7f800000);

  bool active = false;
  float e0 = 0.f, e1 = 0.f, e2 = 0.f, f0 = 0.f, f1 = 0.f, f2 = 0.f;
  float i0 = 0.f, i1 = 0.f, i2 = 0.f, k0 = kInf, k1 = kInf, k2 = kInf;
  int c0 = 0, c1 = 0, c2 = 0, dL0 = 0, dL1 = 0, dL2 = 0, left = 0;
  bool x0 = false, x1 = false, x2 = false;
  uint32_t L = 0;

  if (p < n) {
    const float4 q = __ldg(pts + p);
    float g0, g1, g2;
    if (transform_point(sp, q, g0, g1, g2)) {
      const int E0 = (int)floorf(g0), E1 = (int)floorf(g1), E2 = (int)floorf(g2);
      const int strideY = d.nz * d.nx;
      // endpoint occupancy (O4/O6: occupied iff hits >= 1)
      if ((unsigned)E0 < (unsigned)d.nx && (unsigned)E1 < (unsigned)d.ny &&
          (unsigned)E2 < (unsigned)d.nz) {
        const uint32_t LE = (uint32_t)(E2 + d.nz * E0 + strideY * E1);
        atomicOr(bits + (LE >> 5), 1u << (LE & 31));
      }
      int r0, r1, r2;
      bool fin = true;
      axis_setup(sp.S[0], E0, g0, s0, d.nx, d.nz, e0, f0, i0, k0, c0, dL0, x0, r0, fin);
      axis_setup(sp.S[1], E1, g1, s1, d.ny, strideY, e1, f1, i1, k1, c1, dL1, x1, r1, fin);
      axis_setup(sp.S[2], E2, g2, s2, d.nz, 1, e2, f2, i2, k2, c2, dL2, x2, r2, fin);
      L = (uint32_t)(sp.S[2] + d.nz * sp.S[0] + strideY * sp.S[1]);
      // steps until E when no axis exits the grid; otherwise the exit ends it
      // (a walk never takes more than nx+ny+nz in-grid steps: hard cap)
      left = (x0 || x1 || x2) ? d.nx + d.ny + d.nz : r0 + r1 + r2;
      active = (r0 | r1 | r2) != 0;  // the sensor voxel is in the grid (host check)
      if (active && !fin) {
        const int S[3] = {sp.S[0], sp.S[1], sp.S[2]}, E[3] = {E0, E1, E2};
        const float g[3] = {g0, g1, g2}, s[3] = {s0, s1, s2};
        walk_exact(S, E, g, s, d, miss);
        active = false;
      }
    }
  }

  const unsigned after = 0xfffffffeu << lane;  // lanes above this one
  unsigned act = __ballot_sync(0xffffffffu, active);
  while (act) {
    // Merge equal voxels of adjacent lanes: one atomic per run of lanes.
    const uint32_t key = active ? L : 0xffffffffu;
    const uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
    const bool head = active && (lane == 0 || prev != key);
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    const uint32_t cnt = (uint32_t)(__clz(__brev((heads | ~act) & after)) - lane);
    asm volatile(
        "{ .reg .pred p; setp.ne.u32 p, %2, 0;\n\t"
        "@p red.relaxed.gpu.global.add.u32 [%0], %1; }" ::"l"(miss + L),
        "r"(cnt), "r"((uint32_t)head)
        : "memory");
    // One DDA step for every lane; inactive lanes compute values that are
    // never emitted (`active` only goes from true to false).
    const bool l10 = k1 < k0;
    const float b01 = l10 ? k1 : k0;
    const bool u2 = k2 < b01;
    const bool u1 = l10 && !u2;
    const bool u0 = !l10 && !u2;
    const int cs = u2 ? c2 : (u1 ? c1 : c0);
    const bool xs = u2 ? x2 : (u1 ? x1 : x0);
    const bool out = xs && cs == 0;  // this step would leave the grid
    e0 = u0 ? __fadd_rn(e0, f0) : e0;
    e1 = u1 ? __fadd_rn(e1, f1) : e1;
    e2 = u2 ? __fadd_rn(e2, f2) : e2;
    c0 -= u0;
    c1 -= u1;
    c2 -= u2;
    L += (uint32_t)(u2 ? dL2 : (u1 ? dL1 : dL0));
    // A non-exit axis that used its last step gets 1/d = +-inf: its key
    // (e - s) * inv is then +inf for good (e - s is nonzero with the sign of
    // the step once the axis has moved).
    const bool exh = !xs && cs == 1;
    i0 = (u0 && exh) ? f0 * kInf : i0;
    i1 = (u1 && exh) ? f1 * kInf : i1;
    i2 = (u2 && exh) ? f2 * kInf : i2;
    k0 = __fmul_rn(__fsub_rn(e0, s0), i0);
    k1 = __fmul_rn(__fsub_rn(e1, s1), i1);
    k2 = __fmul_rn(__fsub_rn(e2, s2), i2);
    --left;
    active = active && !out && left != 0;
    act = __ballot_sync(0xffffffffu, active);
  }
}

__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

// popcount of a block's 1024 bitmask words
__global__ void __launch_bounds__(kRankThreads) k_rank_count(const uint32_t* __restrict__ bits,
                                                             int64_t W,
                                                             uint32_t* __restrict__ block_sums) {
  __shared__ uint32_t wsum[kRankThreads / 32];
  const int64_t base = (int64_t)blockIdx.x * kRankWordsPerBlock + threadIdx.x * 4;
  uint32_t c = 0;
  if (base + 3 < W) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(bits + base));
    c = __popc(v.x) + __popc(v.y) + __popc(v.z) + __popc(v.w);
  } else {
    for (int i = 0; i < 4; ++i)
      if (base + i < W) c += __popc(bits[base + i]);
  }
  c = __reduce_add_sync(0xffffffffu, c);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
    for (int i = 0; i < kRankThreads / 32; ++i) t += wsum[i];
    block_sums[blockIdx.x] = t;
  }
}

// exclusive scan of the block sums (one CTA); total -> *total
__global__ void __launch_bounds__(1024) k_rank_scan(uint32_t* __restrict__ sums, int64_t nblk,
                                                    uint32_t* __restrict__ total) {
  __shared__ uint32_t wsum[32];
  __shared__ uint32_t carry;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < nblk; base += 1024) {
    const int64_t i = base + threadIdx.x;
    const uint32_t v = i < nblk ? sums[i] : 0u;
    const uint32_t inc = warp_incl_scan(v, lane);
    if (lane == 31) wsum[wid] = inc;
    __syncthreads();
    if (wid == 0) {
      const uint32_t w = wsum[lane];
      wsum[lane] = warp_incl_scan(w, lane) - w;
    }
    __syncthreads();
    const uint32_t excl = carry + wsum[wid] + inc - v;
    if (i < nblk) sums[i] = excl;
    __syncthreads();
    if (threadIdx.x == 1023) carry = excl + v;
    __syncthreads();
  }
  if (threadIdx.x == 0) *total = carry;
}

// Block-local per-word prefix of the tile's 1024 words into smem; returns
// nothing, fills spre[] (absolute word prefix) and sbits[].
__device__ __forceinline__ void tile_prefix(const uint32_t* __restrict__ bits, int64_t W,
                                            uint32_t boff, uint32_t* sbits, uint32_t* spre,
                                            uint32_t* wsum) {
  const int t = threadIdx.x, lane = t & 31, wid = t >> 5;
  const int64_t base = (int64_t)blockIdx.x * kRankWordsPerBlock + t * 4;
  uint32_t w4[4];
  if (base + 3 < W) {
    const uint4 v = __ldg(reinterpret_cast<const uint4*>(bits + base));
    w4[0] = v.x;
    w4[1] = v.y;
    w4[2] = v.z;
    w4[3] = v.w;
  } else {
    for (int i = 0; i < 4; ++i) w4[i] = (base + i < W) ? bits[base + i] : 0u;
  }
  const uint32_t c0 = __popc(w4[0]), c1 = __popc(w4[1]), c2 = __popc(w4[2]), c3 = __popc(w4[3]);
  const uint32_t tsum = c0 + c1 + c2 + c3;
  const uint32_t inc = warp_incl_scan(tsum, lane);
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const uint32_t w = lane < kRankThreads / 32 ? wsum[lane] : 0u;
    const uint32_t e = warp_incl_scan(w, lane) - w;
    if (lane < kRankThreads / 32) wsum[lane] = e;
  }
  __syncthreads();
  const uint32_t p0 = boff + wsum[wid] + inc - tsum;
  sbits[4 * t + 0] = w4[0];
  sbits[4 * t + 1] = w4[1];
  sbits[4 * t + 2] = w4[2];
  sbits[4 * t + 3] = w4[3];
  spre[4 * t + 0] = p0;
  spre[4 * t + 1] = p0 + c0;
  spre[4 * t + 2] = p0 + c0 + c1;
  spre[4 * t + 3] = p0 + c0 + c1 + c2;
  __syncthreads();
}

__device__ __forceinline__ void store_prefix(uint32_t* __restrict__ wprefix, int64_t W,
                                             const uint32_t* spre) {
  const int t = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * kRankWordsPerBlock + t * 4;
  if (base + 3 < W) {
    *reinterpret_cast<uint4*>(wprefix + base) =
        make_uint4(spre[4 * t], spre[4 * t + 1], spre[4 * t + 2], spre[4 * t + 3]);
  } else {
    for (int i = 0; i < 4; ++i)
      if (base + i < W) wprefix[base + i] = spre[4 * t + i];
  }
}

// O6 in place: buf[L] holds the miss count; becomes rank (occupied) or
// -1 - min(N_m, 2^30) (empty).  Occupied rows get {0, misses, 0xFFFFFFFF, 0, 0, 0}
// for the endpoint pass to accumulate into.  One thread per 4 voxels (one
// 16-byte load + store); rank from the absolute per-word prefix.
__global__ void __launch_bounds__(256) k_finalize(int32_t* __restrict__ buf,
                                                  const uint32_t* __restrict__ bits,
                                                  const uint32_t* __restrict__ wprefix,
                                                  gvom_voxel* __restrict__ data, const Dims d) {
  const int64_t L = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4;
  if (L >= d.V) return;
  const uint32_t bw = __ldg(bits + (L >> 5));
  const uint32_t pre = __ldg(wprefix + (L >> 5));
  const bool vec = (L + 3 < d.V);
  uint32_t m[4];
  if (vec) {
    const uint4 v = __ldcs(reinterpret_cast<const uint4*>(buf + L));
    m[0] = v.x;
    m[1] = v.y;
    m[2] = v.z;
    m[3] = v.w;
  } else {
    for (int j = 0; j < 4; ++j) m[j] = (L + j < d.V) ? (uint32_t)buf[L + j] : 0u;
  }
  int32_t o[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int bit = (int)((L + j) & 31);
    if ((bw >> bit) & 1u) {
      const uint32_t rank = pre + __popc(bw & ((1u << bit) - 1u));
      o[j] = (int32_t)rank;
      uint4* row = reinterpret_cast<uint4*>(data + rank);
      row[0] = make_uint4(0u, m[j], 0xffffffffu, 0u);
      row[1] = make_uint4(0u, 0u, 0u, 0u);
    } else {
      const uint32_t nm = m[j] < kMissSat ? m[j] : kMissSat;
      o[j] = -1 - (int32_t)nm;
    }
  }
  if (vec) {
    *reinterpret_cast<int4*>(buf + L) = make_int4(o[0], o[1], o[2], o[3]);
  } else {
    for (int j = 0; j < 4; ++j)
      if (L + j < d.V) buf[L + j] = o[j];
  }
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

// Zero two regions in one launch (the slot's LUT-as-miss-grid and bitmask).
__global__ void __launch_bounds__(256) k_zero2(uint4* __restrict__ a, int64_t na16,
                                               uint4* __restrict__ b, int64_t nb16) {
  const uint4 z = make_uint4(0u, 0u, 0u, 0u);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < na16 + nb16; i += stride) {
    if (i < na16)
      __stcs(a + i, z);
    else
      __stcs(b + (i - na16), z);
  }
}

// per-word absolute prefix only (merged-map export)
__global__ void __launch_bounds__(kRankThreads) k_prefix_only(const uint32_t* __restrict__ bits,
                                                              uint32_t* __restrict__ wprefix,
                                                              const uint32_t* __restrict__ boff,
                                                              const Dims d) {
  __shared__ uint32_t sbits[kRankWordsPerBlock];
  __shared__ uint32_t spre[kRankWordsPerBlock];
  __shared__ uint32_t wsum[32];
  tile_prefix(bits, d.W, boff[blockIdx.x], sbits, spre, wsum);
  store_prefix(wprefix, d.W, spre);
}

// O4 per return: hits, min_dz, m1 = sum dz, m2 = sum dz^2 into the data row.
__global__ void __launch_bounds__(256) k_endpoint(const float4* __restrict__ pts, int64_t n,
                                                  int32_t rings, const SensorParams sp,
                                                  const Dims d, const int32_t* __restrict__ lut,
                                                  gvom_voxel* __restrict__ data) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p = point_index(tid, rings);
  if (p >= n) return;
  const float4 q = __ldg(pts + p);
  float g0, g1, g2;
  if (!transform_point(sp, q, g0, g1, g2)) return;
  const int e0 = (int)floorf(g0), e1 = (int)floorf(g1), e2 = (int)floorf(g2);
  if ((unsigned)e0 >= (unsigned)d.nx || (unsigned)e1 >= (unsigned)d.ny ||
      (unsigned)e2 >= (unsigned)d.nz)
    return;
  const int64_t LE = (int64_t)e2 + (int64_t)d.nz * e0 + (int64_t)d.nz * d.nx * e1;
  const int32_t rank = __ldg(lut + LE);
  // qz = floor(f32(g_z * 65536)) is exact (power-of-two scale)
  const int64_t qz = (int64_t)floorf(__fmul_rn(g2, 65536.0f));
  const uint32_t dz = (uint32_t)(qz - 65536ll * e2);
  gvom_voxel* row = data + rank;
  atomicAdd(&row->hits, 1u);
  atomicMin(&row->min_dz, dz);
  atomicAdd(reinterpret_cast<unsigned long long*>(&row->m1), (unsigned long long)dz);
  atomicAdd(reinterpret_cast<unsigned long long*>(&row->m2),
            (unsigned long long)dz * (unsigned long long)dz);
}

inline int64_t point_threads(int64_t n, int32_t rings) {
  if (rings <= 1) return n;
  const int64_t cols = (n + rings - 1) / rings;
  const int64_t tiles = (cols + 31) / 32;
  return tiles * 32 * rings;
}

}  // namespace

cudaError_t launch_raycast(const float4* pts, int64_t n, int32_t rings, const SensorParams& sp,
                           const Dims& d, uint32_t* miss_grid, uint32_t* bits, cudaStream_t st) {
  const int64_t threads = point_threads(n, rings);
  if (threads == 0) return cudaSuccess;
  const int64_t blocks = (threads + 255) / 256;
  k_raycast<<<(unsigned)blocks, 256, 0, st>>>(pts, n, rings, sp, d, miss_grid, bits);
  return cudaGetLastError();
}

cudaError_t launch_rank_count(const uint32_t* bits, const Dims& d, uint32_t* block_sums,
                              cudaStream_t st) {
  k_rank_count<<<(unsigned)rank_blocks(d), kRankThreads, 0, st>>>(bits, d.W, block_sums);
  return cudaGetLastError();
}

cudaError_t launch_rank_scan(uint32_t* block_sums, int64_t nblk, uint32_t* total,
                             cudaStream_t st) {
  k_rank_scan<<<1, 1024, 0, st>>>(block_sums, nblk, total);
  return cudaGetLastError();
}

cudaError_t launch_finalize(int32_t* lut_inplace, const uint32_t* bits, const uint32_t* wprefix,
                            gvom_voxel* data, const Dims& d, cudaStream_t st) {
  const int64_t threads = (d.V + 3) / 4;
  k_finalize<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(lut_inplace, bits, wprefix, data,
                                                                d);
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

cudaError_t launch_zero2(void* a, size_t abytes, void* b, size_t bbytes, cudaStream_t st) {
  const int64_t n = (int64_t)(abytes / 16 + bbytes / 16);
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  k_zero2<<<(unsigned)blocks, 256, 0, st>>>((uint4*)a, (int64_t)(abytes / 16), (uint4*)b,
                                            (int64_t)(bbytes / 16));
  return cudaGetLastError();
}

cudaError_t launch_prefix_only(const uint32_t* bits, uint32_t* wprefix, const uint32_t* block_off,
                               const Dims& d, cudaStream_t st) {
  k_prefix_only<<<(unsigned)rank_blocks(d), kRankThreads, 0, st>>>(bits, wprefix, block_off, d);
  return cudaGetLastError();
}

cudaError_t launch_endpoint(const float4* pts, int64_t n, int32_t rings, const SensorParams& sp,
                            const Dims& d, const int32_t* lut, gvom_voxel* data, cudaStream_t st) {
  const int64_t threads = point_threads(n, rings);
  if (threads == 0) return cudaSuccess;
  const int64_t blocks = (threads + 255) / 256;
  k_endpoint<<<(unsigned)blocks, 256, 0, st>>>(pts, n, rings, sp, d, lut, data);
  return cudaGetLastError();
}

}  // namespace gvom
