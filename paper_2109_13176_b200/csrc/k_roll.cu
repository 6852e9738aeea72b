// k_roll.cu -- the rolling map (SURVEY 8(f) NEXT-3 "rolling in-place map
// (K = inf, toroidal indexing, O(exposed slab) shifts)"; reading B9)
// on sm_100a.
//
// One window map accumulated over every scan since each voxel entered the
// window.  It is stored toroidally in WORLD voxel coordinates: world voxel w
// lives at physical (w_x mod nx, w_y mod ny, w_z mod nz), so moving the window
// moves no data -- only the slabs that enter it are cleared.  Counts are u64
// (a voxel next to the sensor passes every ray of every scan), in separate
// arrays so that a pass-through costs one 8-byte read-modify-write; min_dz is
// kept complemented so that an all-zero workspace is the empty map.
//
//   clear      : zero the entering slabs after a window move (gvom_shift)
//   accumulate : add a scan's frame map (LUT + data rows, built by the usual
//                integrate pipeline) into the window map
//   columns    : O8 on the window map -> the same layer
//                buffers k_columns writes, then k_slope / k_negative as usual
//   export     : the window map in logical (L) order, dense (test / debug)
#include <math.h>

#include "gvom_internal.cuh"

namespace gvom {

namespace {

__device__ __forceinline__ int pmod(int64_t a, int n) {
  const int r = (int)(a % n);
  return r < 0 ? r + n : r;
}

__device__ __forceinline__ int wrap(int v, int n) { return v >= n ? v - n : v; }

// physical index of logical voxel (x, y, z) of the window at origin o
__device__ __forceinline__ int64_t roll_phys(const Dims& d, const RollGrid& g, int x, int y,
                                             int z) {
  const int px = wrap(x + g.xo, d.nx), py = wrap(y + g.yo, d.ny), pz = wrap(z + g.zo, d.nz);
  return (int64_t)pz + (int64_t)d.nz * ((int64_t)px + (int64_t)d.nx * py);
}

// Clear the voxels of the window whose coordinate on `axis` (0 x, 1 y, 2 z)
// is one of the world values w0 .. w0 + cnt - 1 (an entering slab).
__global__ void __launch_bounds__(256) k_roll_clear(const RollGrid g, const Dims d, int axis,
                                                    int64_t w0, int cnt) {
  const int n[3] = {d.nx, d.ny, d.nz};
  const int a1 = axis == 0 ? 1 : 0, a2 = axis == 2 ? 1 : 2;  // the other two axes
  const int64_t per = (int64_t)n[a1] * n[a2];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= per * cnt) return;
  const int64_t o[3] = {g.ox, g.oy, g.oz};
  int p[3];
  p[axis] = pmod(w0 + i / per, n[axis]);
  const int64_t r = i % per;
  p[a1] = pmod(o[a1] + r % n[a1], n[a1]);
  p[a2] = pmod(o[a2] + r / n[a1], n[a2]);
  const int64_t P = (int64_t)p[2] + (int64_t)d.nz * ((int64_t)p[0] + (int64_t)d.nx * p[1]);
  g.hits[P] = 0;
  g.misses[P] = 0;
  g.m1[P] = 0;
  g.m2[P] = 0;
  g.nmn[P] = 0;
  atomicAnd(g.bits + (P >> 5), ~(1u << (P & 31)));
}

// Add a frame map (LUT + data rows over the window at origin g.o) into the
// window map.  Every physical voxel receives from exactly one logical voxel,
// so the counts need no atomics; occupancy bits of neighbours share words.
// Four consecutive voxels of an (x, y) row per thread (one 16-byte LUT load)
// when the row length allows it.
__device__ __forceinline__ void roll_add(const RollGrid& g, int64_t P, int32_t v,
                                         const gvom_voxel* __restrict__ data) {
  if (v >= 0) {
    const gvom_voxel s = data[v];
    g.hits[P] += s.hits;
    g.misses[P] += s.misses;
    g.m1[P] += s.m1;
    g.m2[P] += s.m2;
    g.nmn[P] = max(g.nmn[P], ~s.min_dz);
    atomicOr(g.bits + (P >> 5), 1u << (P & 31));
  } else if (v != -1) {
    g.misses[P] += (uint64_t)(-1 - (int64_t)v);
  }
}

template <int kVec>
__global__ void __launch_bounds__(256) k_roll_accumulate(const RollGrid g, const Dims d,
                                                         const int32_t* __restrict__ lut,
                                                         const gvom_voxel* __restrict__ data) {
  const int row = d.nx * d.nz;  // < 2^31 (gvom_create)
  const int j0 = (blockIdx.x * blockDim.x + threadIdx.x) * kVec;
  const int y = blockIdx.y;
  if (j0 >= row) return;
  int32_t v[kVec];
  if (kVec == 4) {
    const int4 q = __ldcs(reinterpret_cast<const int4*>(lut + (int64_t)y * row + j0));
    v[0] = q.x;
    v[1] = q.y;
    v[2] = q.z;
    v[3] = q.w;
  } else {
    v[0] = __ldcs(lut + (int64_t)y * row + j0);
  }
  bool any = false;
#pragma unroll
  for (int t = 0; t < kVec; ++t) any |= v[t] != -1;
  if (!any) return;  // empty, no ray passed
  const int x = j0 / d.nz, z0 = j0 - x * d.nz;
  const int64_t col = (int64_t)d.nz * ((int64_t)wrap(x + g.xo, d.nx) +
                                       (int64_t)d.nx * wrap(y + g.yo, d.ny));
  int pz = wrap(z0 + g.zo, d.nz);
#pragma unroll
  for (int t = 0; t < kVec; ++t) {  // kVec divides nz: the group stays in one column
    roll_add(g, col + pz, v[t], data);
    pz = pz + 1 == d.nz ? 0 : pz + 1;
  }
}

// O8 on the window map, one thread per column: z* = lowest occupied logical
// z, q_s = 65536 z* + min_dz(z*), the band sums over occupied voxels with
// T_lo <= q - q_s <= T_hi; the same outputs as k_columns (layers, q_s,
// cone-sweep keys and accumulators, point spread).
__global__ void __launch_bounds__(256) k_columns_roll(const RollGrid g, const Dims d,
                                                      const LayerParams lp, const LayerPtrs out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)d.nx * d.ny) return;
  const int x = (int)(c % d.nx), y = (int)(c / d.nx);
  const int px = wrap(x + g.xo, d.nx), py = wrap(y + g.yo, d.ny), zoff = g.zo;
  const int64_t col = (int64_t)d.nz * ((int64_t)px + (int64_t)d.nx * py);
  auto phys = [&](int z) { return col + (z + zoff < d.nz ? z + zoff : z + zoff - d.nz); };
  auto occ = [&](int z) {
    const int64_t P = phys(z);
    return (__ldg(g.bits + (P >> 5)) >> (P & 31)) & 1u;
  };
  int zs = -1;
  for (int z = 0; z < d.nz; ++z) {
    // whole 32-bit words of the column at a time while they are empty
    const int64_t P = phys(z);
    if ((P & 31) == 0 && z + 32 <= d.nz && (z + zoff >= d.nz || z + zoff + 32 <= d.nz) &&
        __ldg(g.bits + (P >> 5)) == 0u) {
      z += 31;
      continue;
    }
    if (occ(z)) {
      zs = z;
      break;
    }
  }
  out.hard[c] = 0;
  out.soft[c] = 0;
  out.nmin[c] = INT32_MAX;
  out.nmax[c] = INT32_MIN;
  const int32_t qv =
      zs < 0 ? kQsUndef : (int32_t)(65536ll * zs + (int64_t)~__ldg(g.nmn + phys(zs)));
  out.qs[c] = qv;
  {
    uint32_t ka, kb;
    neg_keys(qv, lp, ka, kb);
    out.negA[c] = ka;
    out.negB[c] = kb;
    out.negAT[(int64_t)x * d.ny + y] = ka;
    out.negBT[(int64_t)x * d.ny + y] = kb;
  }
  if (zs < 0) {
    out.height[c] = __int_as_float(0x7fc00000);
    out.density[c] = __int_as_float(0x7fc00000);
    out.spread[c] = __int_as_float(0x7fc00000);
    return;
  }
  const int64_t q_s = qv;
  {
    const int64_t P = phys(zs);
    const uint64_t H = __ldg(g.hits + P), M1 = __ldg(g.m1 + P), M2 = __ldg(g.m2 + P);
    const unsigned __int128 num = (unsigned __int128)H * M2 - (unsigned __int128)M1 * M1;
    const double hh = (double)H, sc = lp.res / 65536.0;
    out.spread[c] = (float)((double)num / (hh * hh) * (sc * sc));
  }
  out.height[c] = (float)(((double)(lp.o_z * 65536 + q_s) * lp.res) / 65536.0);
  const int64_t zh = (q_s + lp.T_hi) >> 16;
  const int z_hi = (int)(zh < (int64_t)d.nz - 1 ? zh : (int64_t)d.nz - 1);
  uint64_t SH = 0, SW = 0;
  for (int z = zs; z <= z_hi; ++z) {
    if (!occ(z)) continue;
    const int64_t P = phys(z);
    const int64_t dq = (65536ll * z + (int64_t)~__ldg(g.nmn + P)) - q_s;
    if (dq >= lp.T_lo && dq <= lp.T_hi) {
      const uint64_t h = __ldg(g.hits + P), mi = __ldg(g.misses + P);
      SH += h;
      SW += h + mi;
    }
  }
  if (SH == 0) {
    out.density[c] = 0.0f;
    return;
  }
  out.density[c] = (float)((double)SH / (double)SW);
  if ((uint64_t)65536 * SH >= (uint64_t)lp.tau * SW)
    out.hard[c] = 1;
  else
    out.soft[c] = 1;
}

// the window map in logical order: hits, misses, min_dz, m1, m2 per voxel
__global__ void __launch_bounds__(256) k_roll_export(const RollGrid g, const Dims d,
                                                     uint64_t* __restrict__ hits,
                                                     uint64_t* __restrict__ misses,
                                                     uint32_t* __restrict__ min_dz,
                                                     uint64_t* __restrict__ m1,
                                                     uint64_t* __restrict__ m2) {
  const int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (L >= d.V) return;
  const int z = (int)(L % d.nz), x = (int)((L / d.nz) % d.nx), y = (int)(L / ((int64_t)d.nz * d.nx));
  const int64_t P = roll_phys(d, g, x, y, z);
  hits[L] = g.hits[P];
  misses[L] = g.misses[P];
  m1[L] = g.m1[P];
  m2[L] = g.m2[P];
  min_dz[L] = ~g.nmn[P];
}

}  // namespace

cudaError_t launch_roll_clear(const RollGrid& g, const Dims& d, int axis, int64_t w0, int cnt,
                              cudaStream_t st) {
  const int64_t n[3] = {d.nx, d.ny, d.nz};
  const int64_t per = n[axis == 0 ? 1 : 0] * n[axis == 2 ? 1 : 2];
  const int64_t threads = per * cnt;
  if (threads == 0) return cudaSuccess;
  k_roll_clear<<<(unsigned)((threads + 255) / 256), 256, 0, st>>>(g, d, axis, w0, cnt);
  return cudaGetLastError();
}

cudaError_t launch_roll_accumulate(const RollGrid& g, const Dims& d, const int32_t* lut,
                                   const gvom_voxel* data, cudaStream_t st) {
  const int64_t row = (int64_t)d.nx * d.nz;
  if (d.nz % 4 == 0) {  // rows are whole 16-byte groups of one column each
    const int64_t groups = row / 4;
    k_roll_accumulate<4><<<dim3((unsigned)((groups + 255) / 256), (unsigned)d.ny), 256, 0, st>>>(
        g, d, lut, data);
  } else {
    k_roll_accumulate<1><<<dim3((unsigned)((row + 255) / 256), (unsigned)d.ny), 256, 0, st>>>(
        g, d, lut, data);
  }
  return cudaGetLastError();
}

cudaError_t launch_columns_roll(const RollGrid& g, const Dims& d, const LayerParams& lp,
                                const LayerPtrs& out, cudaStream_t st) {
  const int64_t cells = (int64_t)d.nx * d.ny;
  k_columns_roll<<<(unsigned)((cells + 255) / 256), 256, 0, st>>>(g, d, lp, out);
  return cudaGetLastError();
}

cudaError_t launch_roll_export(const RollGrid& g, const Dims& d, uint64_t* hits, uint64_t* misses,
                               uint32_t* min_dz, uint64_t* m1, uint64_t* m2, cudaStream_t st) {
  k_roll_export<<<(unsigned)((d.V + 255) / 256), 256, 0, st>>>(g, d, hits, misses, min_dz, m1,
                                                               m2);
  return cudaGetLastError();
}

}  // namespace gvom
