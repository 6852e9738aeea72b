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

// O5 stateless key: f32( f32( f32(V + [step>0]) - s ) * inv )
__device__ __forceinline__ float dda_key(int v, int st, float s, float inv) {
  return __fmul_rn(__fsub_rn(__int2float_rn(v + (st > 0 ? 1 : 0)), s), inv);
}

__device__ __forceinline__ int isign(int v) { return (v > 0) - (v < 0); }

__global__ void __launch_bounds__(256) k_raycast(const float4* __restrict__ pts, int64_t n,
                                                 int32_t rings, const SensorParams sp,
                                                 const Dims d, uint32_t* __restrict__ miss,
                                                 uint32_t* __restrict__ bits) {
  const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t p = point_index(tid, rings);
  const int lane = threadIdx.x & 31;

  bool active = false;
  int v0 = 0, v1 = 0, v2 = 0, st0 = 0, st1 = 0, st2 = 0, r0 = 0, r1 = 0, r2 = 0;
  float s0 = sp.b[0], s1 = sp.b[1], s2 = sp.b[2];
  float i0 = 0.f, i1 = 0.f, i2 = 0.f, k0 = 0.f, k1 = 0.f, k2 = 0.f;
  int64_t L = 0;
  const int64_t dLx = d.nz, dLy = (int64_t)d.nz * d.nx;

  if (p < n) {
    const float4 q = __ldg(pts + p);
    float g0, g1, g2;
    if (transform_point(sp, q, g0, g1, g2)) {
      const int e0 = (int)floorf(g0), e1 = (int)floorf(g1), e2 = (int)floorf(g2);
      // endpoint occupancy (O4/O6: occupied iff hits >= 1)
      if ((unsigned)e0 < (unsigned)d.nx && (unsigned)e1 < (unsigned)d.ny &&
          (unsigned)e2 < (unsigned)d.nz) {
        const int64_t LE = (int64_t)e2 + dLx * e0 + dLy * e1;
        atomicOr(bits + (LE >> 5), 1u << (LE & 31));
      }
      v0 = sp.S[0];
      v1 = sp.S[1];
      v2 = sp.S[2];
      st0 = isign(e0 - v0);
      st1 = isign(e1 - v1);
      st2 = isign(e2 - v2);
      r0 = abs(e0 - v0);
      r1 = abs(e1 - v1);
      r2 = abs(e2 - v2);
      if (r0 > 0) {
        i0 = __frcp_rn(__fsub_rn(g0, s0));
        k0 = dda_key(v0, st0, s0, i0);
      }
      if (r1 > 0) {
        i1 = __frcp_rn(__fsub_rn(g1, s1));
        k1 = dda_key(v1, st1, s1, i1);
      }
      if (r2 > 0) {
        i2 = __frcp_rn(__fsub_rn(g2, s2));
        k2 = dda_key(v2, st2, s2, i2);
      }
      L = (int64_t)v2 + dLx * v0 + dLy * v1;
      active = (r0 + r1 + r2) > 0;  // the sensor voxel is in the grid (host check)
    }
  }

  for (;;) {
    const unsigned act = __ballot_sync(0xffffffffu, active);
    if (act == 0u) break;
    // Merge equal voxels of adjacent lanes: one atomic per run.
    const uint32_t key = active ? (uint32_t)L : 0xffffffffu;
    const uint32_t prev = __shfl_up_sync(0xffffffffu, key, 1);
    const bool head = active && (lane == 0 || prev != key);
    const unsigned heads = __ballot_sync(0xffffffffu, head);
    if (head) {
      const unsigned after = ~((2u << lane) - 1u);  // lanes > lane
      const unsigned boundary = (heads | ~act) & after;
      const int next = boundary ? (__ffs(boundary) - 1) : 32;
      atomicAdd(miss + L, (uint32_t)(next - lane));
    }
    if (active) {
      // argmin over axes with remaining steps, ties to the lowest axis (O5)
      int best = -1;
      float bk = 0.f;
      if (r0 > 0) {
        best = 0;
        bk = k0;
      }
      if (r1 > 0 && (best < 0 || k1 < bk)) {
        best = 1;
        bk = k1;
      }
      if (r2 > 0 && (best < 0 || k2 < bk)) best = 2;
      bool inb;
      if (best == 0) {
        v0 += st0;
        --r0;
        L += dLx * st0;
        k0 = dda_key(v0, st0, s0, i0);
        inb = (unsigned)v0 < (unsigned)d.nx;
      } else if (best == 1) {
        v1 += st1;
        --r1;
        L += dLy * st1;
        k1 = dda_key(v1, st1, s1, i1);
        inb = (unsigned)v1 < (unsigned)d.ny;
      } else {
        v2 += st2;
        --r2;
        L += st2;
        k2 = dda_key(v2, st2, s2, i2);
        inb = (unsigned)v2 < (unsigned)d.nz;
      }
      active = inb && (r0 + r1 + r2) > 0;
    }
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
// for the endpoint pass to accumulate into.
__global__ void __launch_bounds__(kRankThreads) k_finalize(int32_t* __restrict__ buf,
                                                           const uint32_t* __restrict__ bits,
                                                           uint32_t* __restrict__ wprefix,
                                                           const uint32_t* __restrict__ block_off,
                                                           gvom_voxel* __restrict__ data,
                                                           const Dims d) {
  __shared__ uint32_t sbits[kRankWordsPerBlock];
  __shared__ uint32_t spre[kRankWordsPerBlock];
  __shared__ uint32_t wsum[32];
  tile_prefix(bits, d.W, block_off[blockIdx.x], sbits, spre, wsum);
  store_prefix(wprefix, d.W, spre);
  const int64_t vbase = (int64_t)blockIdx.x * kRankWordsPerBlock * 32;
  for (int i = threadIdx.x * 4; i < kRankWordsPerBlock * 32; i += kRankThreads * 4) {
    const int64_t L = vbase + i;
    if (L >= d.V) break;
    const bool vec = (L + 3 < d.V);
    uint32_t m[4];
    if (vec) {
      const uint4 v = *reinterpret_cast<const uint4*>(buf + L);
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
      const int l = i + j;
      const uint32_t bw = sbits[l >> 5];
      const int bit = l & 31;
      if ((bw >> bit) & 1u) {
        const uint32_t rank = spre[l >> 5] + __popc(bw & ((1u << bit) - 1u));
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

cudaError_t launch_finalize(int32_t* lut_inplace, const uint32_t* bits, uint32_t* wprefix,
                            const uint32_t* block_off, gvom_voxel* data, const Dims& d,
                            cudaStream_t st) {
  k_finalize<<<(unsigned)rank_blocks(d), kRankThreads, 0, st>>>(lut_inplace, bits, wprefix,
                                                                 block_off, data, d);
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
