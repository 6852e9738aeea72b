// k_slab.cu -- kernels of the multi-GPU slab partition.
//
// A frame's points are sharded across ranks; each rank traces its rays into a
// dense miss grid (k_raycast with bits == nullptr) and emits its in-grid
// returns as (L, dz) records grouped by destination slab (k_ep_count /
// k_ep_write).  The slab owner rebuilds occupancy from the records it
// receives (k_slab_bits + k_tile_scan), finalizes the slab (k_finalize_tiles
// over the slab's tiles) and accumulates the per-return statistics
// (k_endpoint_records).  After the surface rows are all-gathered,
// k_transpose_init prepares the cone sweeps over the whole map.
#include "gvom_device.cuh"

namespace gvom {

namespace {

// in-grid return -> record + destination slab (by row y); false otherwise
__device__ __forceinline__ bool return_record(const SensorParams& sp, const float4 q,
                                              const Dims& d, const SlabBounds& sb, EpRecord& r,
                                              int& dest) {
  float g0, g1, g2;
  if (!transform_point(sp, q, g0, g1, g2)) return false;
  const int e0 = (int)floorf(g0), e1 = (int)floorf(g1), e2 = (int)floorf(g2);
  if ((unsigned)e0 >= (unsigned)d.nx || (unsigned)e1 >= (unsigned)d.ny ||
      (unsigned)e2 >= (unsigned)d.nz)
    return false;
  r.L = (uint32_t)(e2 + d.nz * e0 + d.nz * d.nx * e1);
  const int64_t qz = (int64_t)floorf(__fmul_rn(g2, 65536.0f));
  r.dz = (uint32_t)(qz - 65536ll * e2);
  int lo = 0, hi = sb.P - 1;  // slab with y[r] <= e1 < y[r+1]
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (sb.y[mid] <= e1)
      lo = mid;
    else
      hi = mid - 1;
  }
  dest = lo;
  return true;
}

__global__ void __launch_bounds__(256) k_ep_count(const float4* __restrict__ pts, int64_t n,
                                                  const SensorParams sp, const Dims d,
                                                  const SlabBounds sb,
                                                  uint32_t* __restrict__ counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  EpRecord r;
  int dest = -1;
  if (i < n && !return_record(sp, __ldg(pts + i), d, sb, r, dest)) dest = -1;
  const unsigned peers = __match_any_sync(0xffffffffu, dest);
  if (dest >= 0 && lane == __ffs(peers) - 1) atomicAdd(counts + dest, (uint32_t)__popc(peers));
}

__global__ void __launch_bounds__(256) k_ep_write(const float4* __restrict__ pts, int64_t n,
                                                  const SensorParams sp, const Dims d,
                                                  const SlabBounds sb,
                                                  uint32_t* __restrict__ cursor,
                                                  EpRecord* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  EpRecord r;
  int dest = -1;
  if (i < n && !return_record(sp, __ldg(pts + i), d, sb, r, dest)) dest = -1;
  const unsigned peers = __match_any_sync(0xffffffffu, dest);
  const int leader = __ffs(peers) - 1;
  uint32_t base = 0;
  if (dest >= 0 && lane == leader) base = atomicAdd(cursor + dest, (uint32_t)__popc(peers));
  base = __shfl_sync(0xffffffffu, base, leader);
  if (dest >= 0) out[base + __popc(peers & ((1u << lane) - 1u))] = r;
}

// occupancy bits of the slab from its records; newly set bits counted per tile
__global__ void __launch_bounds__(256) k_slab_bits(const EpRecord* __restrict__ ep, int64_t n,
                                                   uint32_t* __restrict__ bits,
                                                   uint32_t* __restrict__ tile_counts) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  uint32_t tile = 0xffffffffu;
  if (i < n) {
    const uint32_t L = ep[i].L;
    const uint32_t bit = 1u << (L & 31);
    if (!(atomicOr(bits + (L >> 5), bit) & bit)) tile = L >> kTileShift;
  }
  const unsigned peers = __match_any_sync(0xffffffffu, tile);
  if (tile != 0xffffffffu && lane == __ffs(peers) - 1)
    atomicAdd(tile_counts + tile, (uint32_t)__popc(peers));
}


// exclusive offsets of the tile counts in [t0, t1) (relative to t0) and their
// total -> *tc.total; one block, each thread a contiguous chunk
__global__ void __launch_bounds__(1024) k_tile_scan(const TileCounts tc, int64_t t0, int64_t t1) {
  __shared__ uint32_t wsum[32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int64_t nt = t1 - t0;
  const int64_t chunk = (nt + blockDim.x - 1) / blockDim.x;
  const int64_t c0 = t0 + threadIdx.x * chunk, c1 = min(t1, c0 + chunk);
  uint32_t sum = 0;
  for (int64_t i = c0; i < c1; ++i) sum += tc.tile[i];
  const uint32_t inc = warp_incl_scan(sum, lane);
  if (lane == 31) wsum[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    const uint32_t w = lane < nw ? wsum[lane] : 0u;
    const uint32_t e = warp_incl_scan(w, lane) - w;
    if (lane < nw) wsum[lane] = e;
    if (lane == nw - 1) *tc.total = e + w;
  }
  __syncthreads();
  uint32_t run = wsum[wid] + inc - sum;
  for (int64_t i = c0; i < c1; ++i) {
    tc.offset[i] = run;
    run += tc.tile[i];
  }
}

// O4 statistics from routed records (order-independent integer atomics)
__global__ void __launch_bounds__(256) k_endpoint_records(const EpRecord* __restrict__ ep,
                                                          int64_t n,
                                                          const int32_t* __restrict__ lut,
                                                          gvom_voxel* __restrict__ data) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const EpRecord r = ep[i];
  gvom_voxel* row = data + __ldg(lut + r.L);
  atomicAdd(&row->hits, 1u);
  atomicMin(&row->min_dz, r.dz);
  atomicAdd(reinterpret_cast<unsigned long long*>(&row->m1), (unsigned long long)r.dz);
  atomicAdd(reinterpret_cast<unsigned long long*>(&row->m2),
            (unsigned long long)r.dz * (unsigned long long)r.dz);
}

// after the surface all-gather: cone-sweep keys (+ transposed copies) and the
// cone-search accumulators
__global__ void __launch_bounds__(256) k_transpose_init(const Dims d, const LayerParams lp,
                                                        const LayerPtrs out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)d.nx * d.ny) return;
  const int x = (int)(c % d.nx), y = (int)(c / d.nx);
  uint32_t ka, kb;
  neg_keys(out.qs[c], lp, ka, kb);
  out.negA[c] = ka;
  out.negB[c] = kb;
  out.negAT[(int64_t)x * d.ny + y] = ka;
  out.negBT[(int64_t)x * d.ny + y] = kb;
  out.nmin[c] = INT32_MAX;
  out.nmax[c] = INT32_MIN;
}

// occupancy word w and its rank prefix (the rank of its first occupied voxel;
// only read for words with a set bit) from a complete LUT
__global__ void __launch_bounds__(256) k_bits_from_lut(const int32_t* __restrict__ lut,
                                                       uint32_t* __restrict__ bits,
                                                       uint32_t* __restrict__ wprefix,
                                                       const Dims d, uint32_t* meta,
                                                       uint32_t k_total) {
  const int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (w == 0) *meta = k_total;
  if (w >= d.W) return;
  uint32_t m = 0, first = 0;
  const int64_t L0 = w * 32;
  for (int i = 31; i >= 0; --i) {
    if (L0 + i >= d.V) continue;
    const int32_t v = __ldg(lut + L0 + i);
    if (v >= 0) {
      m |= 1u << i;
      first = (uint32_t)v;
    }
  }
  bits[w] = m;
  wprefix[w] = first;
}

inline unsigned blocks_for(int64_t n, int tpb) { return (unsigned)((n + tpb - 1) / tpb); }


// Per-row work of a frame map (slab balancing): row y's pass-throughs + returns
// = sum over its voxels of misses + hits -- for an empty voxel the O6 code
// -1 - N_m, for an occupied one its data row.  One block per row, int4 LUT
// loads, the data rows only behind occupied entries.
__global__ void __launch_bounds__(256) k_row_work(const int32_t* __restrict__ lut,
                                                  const gvom_voxel* __restrict__ data,
                                                  const Dims d, int32_t y0,
                                                  unsigned long long* __restrict__ out) {
  const int64_t row = (int64_t)d.nx * d.nz;
  const int64_t y = (int64_t)y0 + blockIdx.x;
  const int32_t* lr = lut + y * row;
  unsigned long long acc = 0ull;
  auto add = [&](int32_t e) {
    if (e < 0) {
      acc += (unsigned)(-1 - e);
    } else {
      const gvom_voxel& v = data[e];
      acc += (unsigned long long)__ldg(&v.misses) + __ldg(&v.hits);
    }
  };
  if ((row & 3) == 0) {  // rows start 16-byte aligned
    const int4* l4 = reinterpret_cast<const int4*>(lr);
    for (int64_t i = threadIdx.x; i < (row >> 2); i += blockDim.x) {
      const int4 q = __ldcs(l4 + i);
      add(q.x);
      add(q.y);
      add(q.z);
      add(q.w);
    }
  } else {
    for (int64_t i = threadIdx.x; i < row; i += blockDim.x) add(__ldcs(lr + i));
  }
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  __shared__ unsigned long long ws[8];
  if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0ull;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
    out[y] = t;
  }
}

}  // namespace

cudaError_t launch_ep_count(const float4* pts, int64_t n, const SensorParams& sp, const Dims& d,
                            const SlabBounds& sb, uint32_t* counts, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_ep_count<<<blocks_for(n, 256), 256, 0, st>>>(pts, n, sp, d, sb, counts);
  return cudaGetLastError();
}

cudaError_t launch_ep_write(const float4* pts, int64_t n, const SensorParams& sp, const Dims& d,
                            const SlabBounds& sb, uint32_t* cursor, EpRecord* out,
                            cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_ep_write<<<blocks_for(n, 256), 256, 0, st>>>(pts, n, sp, d, sb, cursor, out);
  return cudaGetLastError();
}

cudaError_t launch_slab_bits(const EpRecord* ep, int64_t n, uint32_t* bits, uint32_t* tile_counts,
                             cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_slab_bits<<<blocks_for(n, 256), 256, 0, st>>>(ep, n, bits, tile_counts);
  return cudaGetLastError();
}

cudaError_t launch_tile_scan(const TileCounts& tc, int64_t t_begin, int64_t t_end,
                             cudaStream_t st) {
  k_tile_scan<<<1, 1024, 0, st>>>(tc, t_begin, t_end);
  return cudaGetLastError();
}

cudaError_t launch_endpoint_records(const EpRecord* ep, int64_t n, const int32_t* lut,
                                    gvom_voxel* data, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  k_endpoint_records<<<blocks_for(n, 256), 256, 0, st>>>(ep, n, lut, data);
  return cudaGetLastError();
}

cudaError_t launch_bits_from_lut(const int32_t* lut, uint32_t* bits, uint32_t* wprefix,
                                 const Dims& d, uint32_t* meta, uint32_t k_total, cudaStream_t st) {
  k_bits_from_lut<<<blocks_for(d.W, 256), 256, 0, st>>>(lut, bits, wprefix, d, meta, k_total);
  return cudaGetLastError();
}

cudaError_t launch_transpose_init(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                                  cudaStream_t st) {
  k_transpose_init<<<blocks_for((int64_t)d.nx * d.ny, 256), 256, 0, st>>>(d, lp, out);
  return cudaGetLastError();
}

cudaError_t launch_row_work(const int32_t* lut, const gvom_voxel* data, const Dims& d, int32_t y0,
                            int32_t y1, unsigned long long* out, cudaStream_t st) {
  if (y1 <= y0) return cudaSuccess;
  k_row_work<<<(unsigned)(y1 - y0), 256, 0, st>>>(lut, data, d, y0, out);
  return cudaGetLastError();
}

}  // namespace gvom
