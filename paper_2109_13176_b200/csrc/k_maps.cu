// k_maps.cu -- map processing (section III.D) on sm_100a.
//
//   columns : shift + merge of the K buffer maps fused with the column reduce
//             (height P:112, obstacle band density / hard / soft P:114).  Reads
//             only what the column needs: per-slot occupancy bits to find the
//             surface voxel and the band, data rows / LUT cells of the band.
//   slope   : N x N least-squares plane, exact int64 normal equations, double
//             finish
//   negative: 4-cone Chebyshev-ring search over undefined cells
//   merge_* : full combined voxel map (LUT + data) for export
#include <math.h>
#include <stdlib.h>

#include "gvom_internal.cuh"

namespace gvom {

namespace {

// 32 occupancy bits of column `colbase` (= nz * column index) for z in
// [z0, z0+32), restricted to [0, nz); bit i <-> z0 + i.
__device__ __forceinline__ uint32_t col_bits32(const uint32_t* __restrict__ bits, int64_t W,
                                               int64_t colbase, int z0, int nz) {
  const int lo = max(z0, 0), hi = min(z0 + 32, nz);
  if (lo >= hi) return 0u;
  const int64_t p = colbase + lo;
  const int64_t w = p >> 5;
  const int sh = (int)(p & 31);
  uint32_t v = __ldg(bits + w) >> sh;
  if (sh != 0 && w + 1 < W) v |= __ldg(bits + w + 1) << (32 - sh);
  const int nb = hi - lo;
  if (nb < 32) v &= (1u << nb) - 1u;
  return v << (lo - z0);
}

// Occupied voxel of a buffer map -> its data row index (rank in L order).
__device__ __forceinline__ bool slot_rank(const SlotView& s, int64_t L, uint32_t& rank) {
  const int64_t w = L >> 5;
  const int bit = (int)(L & 31);
  const uint32_t bw = __ldg(s.bits + w);
  if (!((bw >> bit) & 1u)) return false;
  rank = __ldg(s.wprefix + w) + __popc(bw & ((1u << bit) - 1u));
  return true;
}

// Segmented (within groups of 2^lg lanes) reductions.
__device__ __forceinline__ uint32_t grp_or(uint32_t v, int lg) {
  for (int o = 1; o < (1 << lg); o <<= 1) v |= __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint64_t grp_add64(uint64_t v, int lg) {
  for (int o = 1; o < (1 << lg); o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ uint32_t grp_min(uint32_t v, int lg) {
  for (int o = 1; o < (1 << lg); o <<= 1) v = min(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// One slot's contribution to output voxel z of this lane's column (O7):
// hits, misses (data row if occupied, -1 - LUT if empty), min_dz.
struct SlotVox {
  uint32_t h, mi, mn;
};
__device__ __forceinline__ SlotVox slot_vox(bool col, const int32_t* __restrict__ lut,
                                            const gvom_voxel* __restrict__ data, int64_t cb,
                                            int uz, int nz) {
  SlotVox r{0u, 0u, 0xffffffffu};
  if (col && (unsigned)uz < (unsigned)nz) {
    const int32_t v = __ldg(lut + cb + uz);
    if (v >= 0) {
      const uint4 row = __ldg(reinterpret_cast<const uint4*>(data + v));
      r.h = row.x;
      r.mi = row.y;
      r.mn = row.z;
    } else {
      r.mi = (uint32_t)(-1 - v);
    }
  }
  return r;
}

// LUT cell of a slot's column at uz; -1 (empty, no misses: contributes
// nothing) when the column is not in the slot's map or uz is off the grid.
__device__ __forceinline__ int32_t lut_cell(bool col, const int32_t* __restrict__ lut,
                                            int64_t cb, int uz, int nz) {
  return (col && (unsigned)uz < (unsigned)nz) ? __ldg(lut + cb + uz) : -1;
}
// The voxel of a LUT cell: data row if occupied, else its miss count.
__device__ __forceinline__ SlotVox cell_vox(int32_t v, const gvom_voxel* __restrict__ data) {
  SlotVox r{0u, 0u, 0xffffffffu};
  if (v >= 0) {
    const uint4 row = __ldg(reinterpret_cast<const uint4*>(data + v));
    r.h = row.x;
    r.mi = row.y;
    r.mn = row.z;
  } else {
    r.mi = (uint32_t)(-1 - v);
  }
  return r;
}

// The column's outputs (lane 0 of its group): q_s and the cone-sweep keys,
// height, point spread (NEXT-3), band density and hard / soft.
__device__ __forceinline__ void write_column(const LayerPtrs& out, const LayerParams& lp,
                                             const Dims& d, int64_t c, int x, int y, int zs,
                                             int64_t q_s, uint64_t sh, uint64_t s1, uint64_t s2,
                                             uint64_t SH, uint64_t SW) {
  out.hard[c] = 0;
  out.soft[c] = 0;
  out.nmin[c] = INT32_MAX;
  out.nmax[c] = INT32_MIN;
  const int32_t qv = zs < 0 ? kQsUndef : (int32_t)q_s;
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
  {
    const unsigned __int128 num = (unsigned __int128)sh * s2 - (unsigned __int128)s1 * s1;
    const double hh = (double)sh, sc = lp.res / 65536.0;
    out.spread[c] = (float)((double)num / (hh * hh) * (sc * sc));
  }
  out.height[c] = (float)(((double)(lp.o_z * 65536 + q_s) * lp.res) / 65536.0);
  if (SH == 0) {
    out.density[c] = 0.0f;
  } else {
    out.density[c] = (float)((double)SH / (double)SW);
    if (65536ull * SH >= (uint64_t)lp.tau * SW)
      out.hard[c] = 1;
    else
      out.soft[c] = 1;
  }
}

// O7 + O8 fused.  2^lg lanes per output column, lane k <-> buffer map k
// (32 >> lg columns per warp).  Per column:
//   z*   : lowest z occupied in any map (OR of the maps' shifted occupancy
//          bits), mn(z*) = min over maps -> q_s.
//   band : voxels strictly between z_lo = (q_s+T_lo)>>16 and z_hi =
//          (q_s+T_hi)>>16 are in [T_lo, T_hi] whatever their min_dz, so each
//          lane sums its own map's hits / hits+misses over them with no
//          cross-lane traffic; only the two edge voxels need the merged
//          min_dz (a group min).  One group sum at the end.
// k_columns' min resident blocks per SM: 6 (40 registers, 16 bytes spilled)
// gives 888 resident blocks instead of 740 for a grid of 1024 (c2) -- the
// second partial wave shrinks: c2 columns 28.0 vs 29.0 us, c4 57.0 vs 63.4 us
// (instrumented, same box); 8 (32 registers) spills more and gains less
#ifndef GVOM_COL_MINB
#define GVOM_COL_MINB 6
#endif
template <bool kEarlyEdges>
__global__ void __launch_bounds__(256, GVOM_COL_MINB) k_columns(const __grid_constant__ SlotSet ss, const Dims d,
                                                 const LayerParams lp, const LayerPtrs out,
                                                 int64_t cbeg, int64_t cells) {
  const int lane = threadIdx.x & 31;
  const int lg = ss.kp_log2;
  const int k = lane & ((1 << lg) - 1);
  const int64_t c0 = cbeg + ((((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) << (5 - lg));
  if (c0 >= cells) return;  // whole warp past the end (cells = end of the range)
  const int64_t c = c0 + (lane >> lg);
  const bool cvalid = c < cells;
  const int x = cvalid ? (int)(c % d.nx) : 0, y = cvalid ? (int)(c / d.nx) : 0;
  bool col = false;
  int64_t cb = 0;
  int dz = 0;
  const uint32_t* bits = nullptr;
  const int32_t* lut = nullptr;
  const gvom_voxel* data = nullptr;
  if (cvalid && k < ss.K) {
    const SlotView& s = ss.s[k];
    const int sx = x + s.dx, sy = y + s.dy;
    if ((unsigned)sx < (unsigned)d.nx && (unsigned)sy < (unsigned)d.ny) {
      col = true;
      cb = (int64_t)d.nz * ((int64_t)sx + (int64_t)d.nx * sy);
      dz = s.dz;
      const int64_t dp = peer_delta(ss.pm, sy);  // the row's owner (slab partition)
      bits = rebase(s.bits, dp);
      lut = rebase(s.lut, dp);
      data = rebase(s.data, dp);
    }
  }
  // ---- z*: merged occupancy, 32 z at a time; keep a 64-z window from the
  // chunk holding z* ----
  int zs = -1, zc = 0;
  uint64_t occ = 0;
  for (int z0 = 0; z0 < d.nz; z0 += 32) {
    uint32_t m = col ? col_bits32(bits, d.W, cb, z0 + dz, d.nz) : 0u;
    m = grp_or(m, lg);
    if (zs >= 0) {
      if (z0 == zc + 32) occ |= (uint64_t)m << 32;  // the chunk after z*'s
    } else if (m) {
      zs = z0 + __ffs(m) - 1;
      zc = z0;
      occ = m;
    }
    if (__all_sync(0xffffffffu, zs >= 0 ? z0 >= zc + 32 : !cvalid)) break;
  }
  // ---- the surface voxel: its whole row (counts + moments) in one go ----
  SlotVox v0{0u, 0u, 0xffffffffu};
  uint64_t sh = 0, s1 = 0, s2 = 0;  // moments (point spread, NEXT-3)
  if (col && zs >= 0 && (unsigned)(zs + dz) < (unsigned)d.nz) {
    const int32_t r0 = __ldg(lut + cb + zs + dz);
    if (r0 >= 0) {
      const uint4 a = __ldg(reinterpret_cast<const uint4*>(data + r0));
      const ulonglong2 mm = __ldg(reinterpret_cast<const ulonglong2*>(data + r0) + 1);
      v0 = SlotVox{a.x, a.y, a.z};
      sh = a.x;
      s1 = mm.x;
      s2 = mm.y;
    } else {
      v0.mi = (uint32_t)(-1 - r0);
    }
  }
  const uint32_t mn0 = grp_min(v0.mn, lg);
  sh = grp_add64(sh, lg);
  s1 = grp_add64(s1, lg);
  s2 = grp_add64(s2, lg);
  const int64_t q_s = 65536ll * zs + (int64_t)mn0;
  const int z_lo = (int)((q_s + lp.T_lo) >> 16);
  const int64_t zh = (q_s + lp.T_hi) >> 16;
  const int z_hi = (int)(zh < (int64_t)d.nz - 1 ? zh : (int64_t)d.nz - 1);
  // occupied in the merged map (any buffer map): from the 64-z bit window
  // above z*'s chunk, else (a band wider than the window, not in the shipped
  // configs) from the maps' LUT cells
  auto occz = [&](int z) -> bool {
    const int rel = z - zc;
    if (rel >= 0 && rel < 64) return (occ >> rel) & 1ull;
    for (int kk = 0; kk < ss.K; ++kk) {
      const SlotView& s = ss.s[kk];
      const int sx = x + s.dx, sy = y + s.dy, uz = z + s.dz;
      if ((unsigned)sx < (unsigned)d.nx && (unsigned)sy < (unsigned)d.ny &&
          (unsigned)uz < (unsigned)d.nz &&
          __ldg(rebase(s.lut, peer_delta(ss.pm, sy)) +
                (int64_t)d.nz * ((int64_t)sx + (int64_t)d.nx * sy) + uz) >= 0)
        return true;
    }
    return false;
  };
  uint64_t SH = 0, SW = 0;
  // edge voxels z_lo and z_hi need the merged min_dz; an edge voxel that no
  // map occupies contributes nothing and is not loaded.  Their LUT cells and
  // rows are loaded first, so they are in flight with the interior band's
  const bool use0 = zs >= 0 && z_lo <= z_hi && z_lo >= zs && occz(z_lo);
  const bool use1 = zs >= 0 && z_hi >= zs && z_hi != z_lo && occz(z_hi);
  SlotVox ve0{0u, 0u, 0xffffffffu}, ve1{0u, 0u, 0xffffffffu};
  if (kEarlyEdges) {
    const int32_t le0 = use0 ? lut_cell(col, lut, cb, z_lo + dz, d.nz) : -1;
    const int32_t le1 = use1 ? lut_cell(col, lut, cb, z_hi + dz, d.nz) : -1;
    if (use0) ve0 = cell_vox(le0, data);
    if (use1) ve1 = cell_vox(le1, data);
  }
  if (zs >= 0) {
    // interior band voxels: certainly in the band when occupied
    const int rlo = z_lo + 1 - zc, rhi = z_hi - zc;  // interior rel range [rlo, rhi)
    if (rlo >= 0 && rhi <= 64) {
      // occupied interior voxels four at a time: their LUT cells, then their
      // rows, all in flight together
      uint64_t mask = rlo < rhi ? occ & ((rhi >= 64 ? ~0ull : (1ull << rhi) - 1ull) &
                                         ~((1ull << rlo) - 1ull))
                                : 0ull;
      while (mask) {
        int32_t lv[4];
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          lv[t] = -1;
          if (mask) {
            const int z = zc + __ffsll((long long)mask) - 1;
            mask &= mask - 1;
            lv[t] = lut_cell(col, lut, cb, z + dz, d.nz);
          }
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const SlotVox v = cell_vox(lv[t], data);
          SH += v.h;
          SW += (uint64_t)v.h + v.mi;
        }
      }
    } else {  // band beyond the 64-z window (not in the shipped configs)
      for (int z = z_lo + 1; z < z_hi; ++z) {
        if (!occz(z)) continue;
        const SlotVox v = slot_vox(col, lut, data, cb, z + dz, d.nz);
        SH += v.h;
        SW += (uint64_t)v.h + v.mi;
      }
    }
  }
  // the edge voxels: in the band iff their merged min_dz puts them there
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int z = e == 0 ? z_lo : z_hi;
    const bool use = e == 0 ? use0 : use1;
    const SlotVox v = kEarlyEdges ? (e == 0 ? ve0 : ve1)
                                  : (use ? slot_vox(col, lut, data, cb, z + dz, d.nz)
                                         : SlotVox{0u, 0u, 0xffffffffu});
    const uint32_t mn = grp_min(v.mn, lg);
    if (use && mn != 0xffffffffu) {
      const int64_t dq = (65536ll * z + (int64_t)mn) - q_s;
      if (dq >= lp.T_lo && dq <= lp.T_hi) {
        SH += v.h;
        SW += (uint64_t)v.h + v.mi;
      }
    }
  }
  SH = grp_add64(SH, lg);
  SW = grp_add64(SW, lg);
  if (k != 0 || !cvalid) return;
  write_column(out, lp, d, c, x, y, zs, q_s, sh, s1, s2, SH, SW);
}

__device__ __forceinline__ int64_t det3(int64_t a, int64_t b, int64_t c, int64_t d, int64_t e,
                                        int64_t f, int64_t g, int64_t h, int64_t i) {
  return a * (e * i - f * h) - b * (d * i - f * g) + c * (d * h - e * g);
}

// O7 + O8 fused, three dependent round trips per column: all occupancy bits
// of the column at once (nz <= 64) -> the LUT cells of every merged-occupied
// voxel that can be in the band, z* first (the band lies in [z*, z* + nb],
// nb = (65535 + T_hi) >> 16, whatever min_dz is) -> their rows, four per batch.
// Then q_s from z*'s merged min, and each candidate classified: strictly
// between z_lo and z_hi it is in the band, on z_lo / z_hi its merged min_dz
// decides (the rule of k_columns, which issues the band and edge loads only
// after z*'s row: up to eight round trips).  Host: nb < 32 (the 64-z window).
__global__ void __launch_bounds__(256) k_columns_fast(const __grid_constant__ SlotSet ss,
                                                      const Dims d, const LayerParams lp,
                                                      const LayerPtrs out, int64_t cbeg,
                                                      int64_t cells, int nb) {
  const int lane = threadIdx.x & 31;
  const int lg = ss.kp_log2;
  const int k = lane & ((1 << lg) - 1);
  const int64_t c0 = cbeg + ((((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) << (5 - lg));
  if (c0 >= cells) return;  // whole warp past the end
  const int64_t c = c0 + (lane >> lg);
  const bool cvalid = c < cells;
  const int x = cvalid ? (int)(c % d.nx) : 0, y = cvalid ? (int)(c / d.nx) : 0;
  bool col = false;
  int64_t cb = 0;
  int dz = 0;
  const uint32_t* bits = nullptr;
  const int32_t* lut = nullptr;
  const gvom_voxel* data = nullptr;
  if (cvalid && k < ss.K) {
    const SlotView& s = ss.s[k];
    const int sx = x + s.dx, sy = y + s.dy;
    if ((unsigned)sx < (unsigned)d.nx && (unsigned)sy < (unsigned)d.ny) {
      col = true;
      cb = (int64_t)d.nz * ((int64_t)sx + (int64_t)d.nx * sy);
      dz = s.dz;
      const int64_t dp = peer_delta(ss.pm, sy);  // the row's owner (slab partition)
      bits = rebase(s.bits, dp);
      lut = rebase(s.lut, dp);
      data = rebase(s.data, dp);
    }
  }
  // ---- z*: merged occupancy; a 64-z window from z*'s 32-z chunk ----
  int zs = -1, zc = 0;
  uint64_t occ = 0;
  if (d.nz <= 64) {  // both chunks in flight together
    uint32_t m0 = col ? col_bits32(bits, d.W, cb, dz, d.nz) : 0u;
    uint32_t m1 = (col && d.nz > 32) ? col_bits32(bits, d.W, cb, 32 + dz, d.nz) : 0u;
    m0 = grp_or(m0, lg);
    m1 = grp_or(m1, lg);
    occ = ((uint64_t)m1 << 32) | m0;
    if (occ) zs = __ffsll((long long)occ) - 1;
  } else {
    for (int z0 = 0; z0 < d.nz; z0 += 32) {
      uint32_t m = col ? col_bits32(bits, d.W, cb, z0 + dz, d.nz) : 0u;
      m = grp_or(m, lg);
      if (zs >= 0) {
        if (z0 == zc + 32) occ |= (uint64_t)m << 32;
      } else if (m) {
        zs = z0 + __ffs(m) - 1;
        zc = z0;
        occ = m;
      }
      if (__all_sync(0xffffffffu, zs >= 0 ? z0 >= zc + 32 : !cvalid)) break;
    }
  }
  // ---- candidates: merged-occupied z in [z*, z* + nb] (relative to zc) ----
  uint64_t cand = 0;
  if (zs >= 0) {
    const int r = zs - zc;  // < 32, and nb < 32: the window holds them
    cand = (occ >> r) & ((2ull << nb) - 1ull);
    cand <<= r;
  }
  uint64_t SH = 0, SW = 0, sh = 0, s1 = 0, s2 = 0;
  int64_t q_s = 0;
  int z_lo = 0, z_hi = -1;
  bool first = true;
  while (__any_sync(0xffffffffu, cand != 0ull)) {
    int32_t lv[4];
    int zz[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      zz[t] = -1;
      lv[t] = -1;
      if (cand) {
        const int z = zc + __ffsll((long long)cand) - 1;
        cand &= cand - 1;
        zz[t] = z;
        lv[t] = lut_cell(col, lut, cb, z + dz, d.nz);
      }
    }
    SlotVox v[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (first && t == 0) {  // z*: the whole row (counts + moments)
        v[0] = SlotVox{0u, 0u, 0xffffffffu};
        if (lv[0] >= 0) {
          const uint4 a = __ldg(reinterpret_cast<const uint4*>(data + lv[0]));
          const ulonglong2 mm = __ldg(reinterpret_cast<const ulonglong2*>(data + lv[0]) + 1);
          v[0] = SlotVox{a.x, a.y, a.z};
          sh = a.x;
          s1 = mm.x;
          s2 = mm.y;
        } else if (zz[0] >= 0) {
          v[0].mi = (uint32_t)(-1 - lv[0]);
        }
      } else {
        v[t] = zz[t] >= 0 ? cell_vox(lv[t], data) : SlotVox{0u, 0u, 0xffffffffu};
      }
    }
    if (first) {
      const uint32_t mn0 = grp_min(v[0].mn, lg);
      sh = grp_add64(sh, lg);
      s1 = grp_add64(s1, lg);
      s2 = grp_add64(s2, lg);
      q_s = 65536ll * zs + (int64_t)mn0;
      z_lo = (int)((q_s + lp.T_lo) >> 16);
      const int64_t zh = (q_s + lp.T_hi) >> 16;
      z_hi = (int)(zh < (int64_t)d.nz - 1 ? zh : (int64_t)d.nz - 1);
      first = false;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const uint32_t mnz = grp_min(v[t].mn, lg);  // the merged min of voxel zz[t]
      const int z = zz[t];
      if (z < 0 || zs < 0) continue;
      bool in = z > z_lo && z < z_hi;
      if (!in && (z == z_lo || z == z_hi) && mnz != 0xffffffffu) {
        const int64_t dq = (65536ll * z + (int64_t)mnz) - q_s;
        in = dq >= lp.T_lo && dq <= lp.T_hi;
      }
      if (in) {
        SH += v[t].h;
        SW += (uint64_t)v[t].h + v[t].mi;
      }
    }
  }
  SH = grp_add64(SH, lg);
  SW = grp_add64(SW, lg);
  if (k != 0 || !cvalid) return;
  write_column(out, lp, d, c, x, y, zs, q_s, sh, s1, s2, SH, SW);
}

// O9: plane fit over the defined in-map cells of the N x N window.
// A 32 x 8 tile of cells plus an r-cell halo of q_s is staged in shared
// memory (kQsUndef = undefined or outside the map), then each thread builds
// the exact int64 normal equations of its window.
constexpr int kSlopeTX = 32, kSlopeTY = 8, kSlopeHalo = 4;  // r <= 4 (N <= 9)
__global__ void __launch_bounds__(kSlopeTX * kSlopeTY) k_slope(const Dims d, const LayerParams lp,
                                                              const LayerPtrs out) {
  constexpr int SW_ = kSlopeTX + 2 * kSlopeHalo, SH_ = kSlopeTY + 2 * kSlopeHalo;
  __shared__ int32_t tile[SH_][SW_ + 1];
  const int r = (lp.slope_window - 1) / 2;
  const int x0 = blockIdx.x * kSlopeTX, y0 = lp.row0 + blockIdx.y * kSlopeTY;
  const int32_t* __restrict__ qs = out.qs;
  for (int i = threadIdx.y * kSlopeTX + threadIdx.x; i < SW_ * SH_; i += kSlopeTX * kSlopeTY) {
    const int ty = i / SW_, tx = i % SW_;
    const int gx = x0 + tx - kSlopeHalo, gy = y0 + ty - kSlopeHalo;
    int32_t q = kQsUndef;
    if ((unsigned)gx < (unsigned)d.nx && (unsigned)gy < (unsigned)d.ny) {
      const int64_t cc = gx + (int64_t)d.nx * gy;
      q = __ldg(qs + cc);
      if (lp.skip_obstacles && (__ldg(out.hard + cc) | __ldg(out.soft + cc))) q = kQsUndef;
    }
    tile[ty][tx] = q;
  }
  __syncthreads();
  const int x = x0 + threadIdx.x, y = y0 + threadIdx.y;
  if (x >= d.nx || y >= lp.row1) return;
  const int64_t c = x + (int64_t)d.nx * y;
  const float qnan = __int_as_float(0x7fc00000);
  const int cx = threadIdx.x + kSlopeHalo, cy = threadIdx.y + kSlopeHalo;
  const int32_t qc = tile[cy][cx];
  if (qc == kQsUndef) {
    out.slope[c] = qnan;
    out.rough[c] = qnan;
    return;
  }
  int32_t n = 0, Su = 0, Sv = 0, Suu = 0, Svv = 0, Suv = 0;
  int64_t Sz = 0, Suz = 0, Svz = 0;
  for (int v = -r; v <= r; ++v)
    for (int u = -r; u <= r; ++u) {
      const int32_t q = tile[cy + v][cx + u];
      if (q == kQsUndef) continue;
      const int64_t z = (int64_t)q - qc;
      n += 1;
      Su += u;
      Sv += v;
      Suu += u * u;
      Svv += v * v;
      Suv += u * v;
      Sz += z;
      Suz += u * z;
      Svz += v * z;
    }
  if (n < lp.min_plane_points) {
    out.slope[c] = qnan;
    out.rough[c] = qnan;
    return;
  }
  const int64_t det = det3(Suu, Suv, Su, Suv, Svv, Sv, Su, Sv, n);
  if (det == 0) {
    out.slope[c] = qnan;
    out.rough[c] = qnan;
    return;
  }
  const int64_t Da = det3(Suz, Suv, Su, Svz, Svv, Sv, Sz, Sv, n);
  const int64_t Db = det3(Suu, Suz, Su, Suv, Svz, Sv, Su, Sz, n);
  const int64_t Dc = det3(Suu, Suv, Suz, Suv, Svv, Svz, Su, Sv, Sz);
  const double a = (double)Da / ((double)det * 65536.0);
  const double b = (double)Db / ((double)det * 65536.0);
  out.slope[c] = (float)atan(sqrt(a * a + b * b));
  double acc = 0.0;
  for (int v = -r; v <= r; ++v)
    for (int u = -r; u <= r; ++u) {
      const int32_t q = tile[cy + v][cx + u];
      if (q == kQsUndef) continue;
      const int64_t z = (int64_t)q - qc;
      const double e = (double)(det * z - Da * u - Db * v - Dc);
      acc += e * e;
    }
  const double sc = lp.res / 65536.0;
  out.rough[c] = (float)(acc / ((double)det * (double)det * (double)n) * (sc * sc));
}

// The same plane fit with the defined cells compacted: a 32 x 8 tile (+ the
// r-cell halo) per 128-thread block; undefined cells are written NaN by the
// thread that classifies them, the defined ones go into a block list (warp
// ballots + a block prefix) that all threads then share, so every lane of a
// warp fits a plane (the per-cell kernel ran ~12 of 32 lanes: undefined
// centres, the double atan's branches).  The finish is atanf of the exact
// normal-equation gradient (within ~2 ulp f32 of the double atan, well inside
// the contract's 1e-4 + 1e-5 |ref|); the nodata decisions are unchanged
// integer tests.
constexpr int kSlope2Threads = 128;                       // 4 warps
constexpr int kSlope2TX = 32, kSlope2TY = 2 * kSlope2Threads / 32;  // 2 rows per warp
__global__ void __launch_bounds__(kSlope2Threads) k_slope_c(const Dims d, const LayerParams lp,
                                                            const LayerPtrs out) {
  constexpr int SW_ = kSlope2TX + 2 * kSlopeHalo, SH_ = kSlope2TY + 2 * kSlopeHalo;
  constexpr int kNW = kSlope2Threads / 32;
  __shared__ int32_t tile[SH_][SW_ + 1];
  __shared__ uint16_t list[kSlope2TX * kSlope2TY];
  __shared__ uint32_t cnt[2 * kNW];
  const int r = (lp.slope_window - 1) / 2;
  const int x0 = blockIdx.x * kSlope2TX, y0 = lp.row0 + blockIdx.y * kSlope2TY;
  const int32_t* __restrict__ qs = out.qs;
  for (int i = threadIdx.x; i < SW_ * SH_; i += kSlope2Threads) {
    const int ty = i / SW_, tx = i % SW_;
    const int gx = x0 + tx - kSlopeHalo, gy = y0 + ty - kSlopeHalo;
    int32_t q = kQsUndef;
    if ((unsigned)gx < (unsigned)d.nx && (unsigned)gy < (unsigned)d.ny) {
      const int64_t cc = gx + (int64_t)d.nx * gy;
      q = __ldg(qs + cc);
      if (lp.skip_obstacles && (__ldg(out.hard + cc) | __ldg(out.soft + cc))) q = kQsUndef;
    }
    tile[ty][tx] = q;
  }
  __syncthreads();
  const float qnan = __int_as_float(0x7fc00000);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned bal[2];
#pragma unroll
  for (int h = 0; h < 2; ++h) {  // warp w classifies rows 2w and 2w + 1
    const int ty = 2 * warp + h, x = x0 + lane, y = y0 + ty;
    const bool inmap = x < d.nx && y < lp.row1;
    const bool def = inmap && tile[ty + kSlopeHalo][lane + kSlopeHalo] != kQsUndef;
    if (inmap && !def) {
      const int64_t c = x + (int64_t)d.nx * y;
      out.slope[c] = qnan;
      out.rough[c] = qnan;
    }
    bal[h] = __ballot_sync(0xffffffffu, def);
    if (lane == 0) cnt[2 * warp + h] = __popc(bal[h]);
  }
  __syncthreads();
  uint32_t total = 0, base[2] = {0u, 0u};
  for (int j = 0; j < 2 * kNW; ++j) {
    const uint32_t v = cnt[j];
    if (j == 2 * warp) base[0] = total;
    if (j == 2 * warp + 1) base[1] = total;
    total += v;
  }
#pragma unroll
  for (int h = 0; h < 2; ++h)
    if ((bal[h] >> lane) & 1u)
      list[base[h] + __popc(bal[h] & ((1u << lane) - 1u))] =
          (uint16_t)((2 * warp + h) * kSlope2TX + lane);
  __syncthreads();
  for (uint32_t it = threadIdx.x; it < total; it += kSlope2Threads) {
    const int li = list[it];
    const int tx = li % kSlope2TX, ty = li / kSlope2TX;
    const int64_t c = (x0 + tx) + (int64_t)d.nx * (y0 + ty);
    const int cx = tx + kSlopeHalo, cy = ty + kSlopeHalo;
    const int32_t qc = tile[cy][cx];
    int32_t n = 0, Su = 0, Sv = 0, Suu = 0, Svv = 0, Suv = 0;
    int64_t Sz = 0, Suz = 0, Svz = 0;
    for (int v = -r; v <= r; ++v)
      for (int u = -r; u <= r; ++u) {
        const int32_t q = tile[cy + v][cx + u];
        if (q == kQsUndef) continue;
        const int64_t z = (int64_t)q - qc;
        n += 1;
        Su += u;
        Sv += v;
        Suu += u * u;
        Svv += v * v;
        Suv += u * v;
        Sz += z;
        Suz += u * z;
        Svz += v * z;
      }
    const int64_t det = det3(Suu, Suv, Su, Suv, Svv, Sv, Su, Sv, n);
    if (n < lp.min_plane_points || det == 0) {
      out.slope[c] = qnan;
      out.rough[c] = qnan;
      continue;
    }
    const int64_t Da = det3(Suz, Suv, Su, Svz, Svv, Sv, Sz, Sv, n);
    const int64_t Db = det3(Suu, Suz, Su, Suv, Svz, Sv, Su, Sz, n);
    const int64_t Dc = det3(Suu, Suv, Suz, Suv, Svv, Svz, Su, Sv, Sz);
    const double a = (double)Da / ((double)det * 65536.0);
    const double b = (double)Db / ((double)det * 65536.0);
    out.slope[c] = atanf((float)sqrt(a * a + b * b));
    double acc = 0.0;
    for (int v = -r; v <= r; ++v)
      for (int u = -r; u <= r; ++u) {
        const int32_t q = tile[cy + v][cx + u];
        if (q == kQsUndef) continue;
        const int64_t z = (int64_t)q - qc;
        const double e = (double)(det * z - Da * u - Db * v - Dc);
        acc += e * e;
      }
    const double sc = lp.res / 65536.0;
    out.rough[c] = (float)(acc / ((double)det * (double)det * (double)n) * (sc * sc));
  }
}

// O10 cone search as a sweep.  For cone +x, let D(x,y) be the first ring k
// (1..K) whose column segment {(x+k, y+t): |t| <= k} holds a defined cell,
// and Mn / Mx the min / max q_s over the defined cells of that ring.  Ring k
// of (x,y) is the union of ring k-1 of the sub-cones with apex (x+1, y-1),
// (x+1, y), (x+1, y+1), so
//   D(x,y) = 1                       if ring 1 (x+1, y-1..y+1) has a defined cell
//          = 1 + min_t D(x+1, y+t)   otherwise (capped: > K = not found),
// and Mn / Mx are the min / max over the sub-cones attaining that minimum
// (their first rings are exactly the pieces of ring D of (x,y)).  With the
// packed keys of neg_keys this is, per key, ONE branch-free min:
//   key(x,y) = min( min_t key_ring1(x+1, y+t),  min_t key(x+1, y+t) + (1 << qb),
//                   not-found ).
// The other cones are the same sweep mirrored / transposed.  Apexes outside
// the map in the cross direction (up to K cells) take part, since their cones
// reach in.  A block sweeps a tile of T lines plus a K-line halo (D <= K
// depends on at most K lines ahead); every found (Mn, Mx) is folded into the
// cell's nmin / nmax with atomics, and k_neg_decide applies
// "max - min > T_neg".  Key lines are streamed into a shared-memory ring by
// 1D TMA bulk copies (cp.async.bulk, mbarrier completion) up to kNegRing lines
// ahead of the sweep; each ring line carries not-found guard cells on both
// sides, so no apex position needs a bounds check.
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar)),
               "r"(count));
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  const uint32_t a = (uint32_t)__cvta_generic_to_shared(bar);
  asm volatile(
      "{ .reg .pred P1;\n"
      "WAIT_%=: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=; }" ::"r"(a),
      "r"(phase)
      : "memory");
}
// bulk-copy global -> shared, completing `bytes` of the transaction count on
// `bar` (the caller announced them with mbarrier.arrive.expect_tx)
__device__ __forceinline__ void tma_copy(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  const uint32_t b = (uint32_t)__cvta_generic_to_shared(bar);
  const uint32_t dsm = (uint32_t)__cvta_generic_to_shared(dst);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(dsm),
      "l"(src), "r"(bytes), "r"(b)
      : "memory");
}

// a ring slot whose line lies outside the map completes its phase empty, so
// every slot's phase parity stays (step / R) & 1
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(
                   (uint32_t)__cvta_generic_to_shared(bar))
               : "memory");
}

// Warp-specialised: the last warp is the producer (TMA bulk copies of the
// ring-1 key lines, R slots ahead, guarded by full/empty mbarriers); the other
// warps are consumers (apex positions strided over them) and sync among
// themselves with a named barrier once per line.
__global__ void __launch_bounds__(1024) k_negative(const Dims d, const LayerParams lp,
                                                        const LayerPtrs out, int T, int R) {
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ __align__(8) uint64_t full[kNegRing], empty[kNegRing];
  const int cone = blockIdx.y;               // 0:+x 1:-x 2:+y 3:-y
  const bool alongx = cone < 2;              // sweep over x (lines = columns)
  const int dir = (cone & 1) ? -1 : 1;       // ring lines lie at p + dir*k
  const int A = alongx ? d.nx : d.ny;        // lines
  const int K = lp.neg_cells;
  const int LB = alongx ? d.ny : d.nx;       // keys per source line
  int c0 = 0, c1 = LB;                       // cross positions held (k_negative_tb)
  if (alongx) {
    c0 = max(0, (lp.row0 - K - 1) & ~3);
    c1 = min(LB, (lp.row1 + K + 1 + 3) & ~3);
  }
  const int B = c1 - c0;                     // cross positions per line
  const int NB = B + 2 * K + 2;              // apex cross positions -K-1 .. B+K
  const int GL = neg_guard_left(K);
  const int LS = neg_line_stride(B, K);      // one key line (A or B keys)
  const int nthr = blockDim.x - 32;          // consumer threads
  const int e0 = alongx ? 0 : lp.row0, e1 = alongx ? d.nx : lp.row1;  // lines emitted
  const uint32_t ONE = 1u << lp.neg_qb;
  const uint32_t NF = (uint32_t)(K + 1) << lp.neg_qb;  // not found
  const uint32_t QM = ONE - 1u;
  uint32_t* ring = sm;                       // [R][2][LS]
  uint32_t* Ap = ring + (size_t)R * 2 * LS;  // sweep state (previous / next line)
  uint32_t* An = Ap + NB;
  uint32_t* Bp = An + NB;
  uint32_t* Bn = Bp + NB;
  const uint32_t* __restrict__ srcA = (alongx ? out.negAT : out.negA) + c0;  // line-contiguous
  const uint32_t* __restrict__ srcB = (alongx ? out.negBT : out.negB) + c0;
  const int p0 = e0 + blockIdx.x * T;        // tile lines [p0, p0+T)
  if (p0 >= e1) return;                      // grid sized for the longest cone
  const int p1 = min(e1, p0 + T);
  int pstart, nsteps;                        // apex lines, in sweep order
  if (dir > 0) {
    pstart = min(A - 1, p1 - 1 + K);
    nsteps = pstart - p0 + 1;
  } else {
    pstart = max(0, p0 - K);
    nsteps = p1 - pstart;
  }
  const bool tma = (B & 3) == 0 && (LB & 3) == 0;  // rows are whole 16-byte chunks
  const uint32_t line_bytes = (uint32_t)B * 4u;
  auto line_of = [&](int st) { return pstart - dir * st + dir; };  // ring-1 line of step st
  for (int i = threadIdx.x; i < NB; i += blockDim.x) {
    Ap[i] = An[i] = NF;  // both buffers: guard apexes are never rewritten
    Bp[i] = Bn[i] = NF;
  }
  // guard cells of every ring line (the TMA writes only [GL, GL + B))
  for (int i = threadIdx.x; i < R * 2 * (LS - B); i += blockDim.x) {
    const int line = i / (LS - B), g = i - line * (LS - B);
    ring[(size_t)line * LS + (g < GL ? g : g + B)] = NF;
  }
  if (threadIdx.x == 0) {
    for (int j = 0; j < R; ++j) {
      mbar_init(&full[j], 1);
      mbar_init(&empty[j], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= nthr) {
    // ---------------- producer warp ----------------
    if (threadIdx.x == nthr) {
      int j = 0;
      uint32_t ph = 0;  // phase parity of the current pass over the ring
      for (int st = 0; st < nsteps; ++st) {
        if (st >= R) mbar_wait(&empty[j], ph ^ 1u);
        const int pl = line_of(st);
        if (tma && pl >= 0 && pl < A) {
          uint32_t* dst = ring + (size_t)j * 2 * LS + GL;
          const uint32_t b = (uint32_t)__cvta_generic_to_shared(&full[j]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                       "r"(2u * line_bytes)
                       : "memory");
          tma_copy(dst, srcA + (int64_t)pl * LB, line_bytes, &full[j]);
          tma_copy(dst + LS, srcB + (int64_t)pl * LB, line_bytes, &full[j]);
        } else {
          mbar_arrive(&full[j]);
        }
        if (++j == R) {
          j = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }
  // ---------------- consumers ----------------
  int j = 0;
  uint32_t ph = 0;  // phase parity of the current pass over the ring
  for (int st = 0; st < nsteps; ++st) {
    const int p = pstart - dir * st;
    const int pl = p + dir;
    const bool inmap = pl >= 0 && pl < A;
    const bool emit = p >= p0 && p < p1;
    uint32_t* la = ring + (size_t)j * 2 * LS;
    uint32_t* lb = la + LS;
    mbar_wait(&full[j], ph);
    if (inmap && !tma) {  // rows not 16-byte multiples: plain loads
      for (int b = threadIdx.x; b < B; b += nthr) {
        la[GL + b] = __ldg(srcA + (int64_t)pl * LB + b);
        lb[GL + b] = __ldg(srcB + (int64_t)pl * LB + b);
      }
      asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    }
    // apex i (cross b = i - K - 1): ring-1 taps b-1..b+1 at la[GL + b - 1 ..]
    const uint32_t* ta = la + GL - K - 2;
    const uint32_t* tb = lb + GL - K - 2;
    for (int i = threadIdx.x + 1; i < NB - 1; i += nthr) {
      uint32_t ka = min(min(Ap[i - 1], Ap[i]), Ap[i + 1]) + ONE;
      uint32_t kb = min(min(Bp[i - 1], Bp[i]), Bp[i + 1]) + ONE;
      if (inmap) {
        ka = min(ka, min(min(ta[i], ta[i + 1]), ta[i + 2]));
        kb = min(kb, min(min(tb[i], tb[i + 1]), tb[i + 2]));
      }
      ka = min(ka, NF);
      kb = min(kb, NF);
      An[i] = ka;
      Bn[i] = kb;
      const int b = i - K - 1, bg = b + c0;
      if (emit && ka < NF && (unsigned)b < (unsigned)B &&
          (!alongx || (bg >= lp.row0 && bg < lp.row1))) {
        const int64_t cell = alongx ? (int64_t)bg * d.nx + p : (int64_t)p * d.nx + bg;
        atomicMin(out.nmin + cell, (int32_t)(ka & QM));
        atomicMax(out.nmax + cell, (int32_t)(QM - (kb & QM)));
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");  // state + slot j consumed
    if (threadIdx.x == 0) mbar_arrive(&empty[j]);
    if (++j == R) {
      j = 0;
      ph ^= 1u;
    }
    uint32_t* t0 = Ap; Ap = An; An = t0;
    t0 = Bp; Bp = Bn; Bn = t0;
  }
}

// O10 with 8 cones (NEXT-3, reading B8): direct search per
// undefined cell (one thread each) over a shared-memory tile of q_s with a
// K-cell halo.  Ring k of the cone at j*45 degrees, in the cone's canonical
// frame (unit vectors a = R^(j/2) (1,0) and b = R^(j/2) (0,1), R the +90
// degree turn):
//   even j: (k, t), |t| <= t_k       (t_k = max t with (t + k)^2 < 2 k^2)
//   odd j : (u, k), t_k < u <= k  and  (k, v), t_k < v < k
// -- straight segments, so whether a ring holds a defined cell is one or two
// O(1) queries on a summed-area table of defined cells; only the first
// non-empty ring of a cone is scanned for its min / max, and a cell with no
// defined cell in its whole (2K+1)^2 square is settled by one query.  (The 8
// rings together are the Chebyshev ring of 8k cells; the oracle tests cone
// membership cell by cell instead.)
__device__ __forceinline__ int neg8_tk(int k) {
  int t = (int)(0.41421356f * (float)k);
  while ((int64_t)(t + 1 + k) * (t + 1 + k) < 2ll * k * k) ++t;
  while (t > 0 && (int64_t)(t + k) * (t + k) >= 2ll * k * k) --t;
  return t;
}

template <int kTile>
__global__ void __launch_bounds__(kTile * kTile) k_negative8(const Dims d, const LayerParams lp,
                                                             const LayerPtrs out) {
  extern __shared__ __align__(16) int32_t tq[];  // [W][W] q_s of tile + halo
  const int K = lp.neg_cells;
  const int W = kTile + 2 * K, W1 = W + 1;
  uint16_t* sat = reinterpret_cast<uint16_t*>(tq + W * W);  // [W1][W1] summed-area table
  uint8_t* tkt = reinterpret_cast<uint8_t*>(sat + W1 * W1);  // t_k, k = 0..K
  const int nthr = kTile * kTile;
  const int gx0 = blockIdx.x * kTile - K, gy0 = blockIdx.y * kTile - K;
  for (int i = threadIdx.x; i < W * W; i += nthr) {
    const int yy = gy0 + i / W, xx = gx0 + i % W;
    tq[i] = ((unsigned)xx < (unsigned)d.nx && (unsigned)yy < (unsigned)d.ny)
                ? __ldg(out.qs + xx + (int64_t)d.nx * yy)
                : kQsUndef;
  }
  for (int k = threadIdx.x; k <= K; k += nthr) tkt[k] = (uint8_t)neg8_tk(k);
  __syncthreads();
  // sat[y][x] = defined cells in [0, x) x [0, y): row prefixes, then columns
  for (int r = threadIdx.x; r < W1; r += nthr) {
    uint16_t n = 0;
    sat[r * W1] = 0;
    for (int x = 0; x < W; ++x) {
      if (r > 0) n += tq[(r - 1) * W + x] != kQsUndef;
      sat[r * W1 + x + 1] = n;
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < W1; c += nthr)
    for (int y = 1; y < W1; ++y) sat[y * W1 + c] += sat[(y - 1) * W1 + c];
  __syncthreads();
  // defined cells in the tile-coordinate rectangle spanned by two corners
  auto rect = [&](int x1, int y1, int x2, int y2) -> int {
    const int lx = min(x1, x2), hx = max(x1, x2) + 1, ly = min(y1, y2), hy = max(y1, y2) + 1;
    return (int)sat[hy * W1 + hx] - sat[hy * W1 + lx] - sat[ly * W1 + hx] + sat[ly * W1 + lx];
  };
  auto seg_minmax = [&](int x1, int y1, int sx, int sy, int n, int32_t& mn, int32_t& mx) {
    for (int i = 0; i < n; ++i) {
      const int32_t q = tq[(y1 + i * sy) * W + (x1 + i * sx)];
      if (q != kQsUndef) {
        mn = min(mn, q);
        mx = max(mx, q);
      }
    }
  };
  const int tx = threadIdx.x % kTile, ty = threadIdx.x / kTile;
  const int x = blockIdx.x * kTile + tx, y = blockIdx.y * kTile + ty;
  if (x >= d.nx || y >= d.ny) return;
  const int cx = tx + K, cy = ty + K;
  const int64_t c = x + (int64_t)d.nx * y;
  if (tq[cy * W + cx] != kQsUndef || rect(cx - K, cy - K, cx + K, cy + K) == 0) {
    out.neg[c] = 0;  // defined, or nothing within reach of any cone
    return;
  }
  int32_t mn = INT32_MAX, mx = INT32_MIN;
  for (int j = 0; j < 8; ++j) {
    int ax = 1, ay = 0, bx = 0, by = 1;
    for (int m = 0; m < j / 2; ++m) {
      const int t0 = ax;
      ax = -ay;
      ay = t0;
      const int t1 = bx;
      bx = -by;
      by = t1;
    }
    for (int k = 1; k <= K; ++k) {
      const int tk = tkt[k];
      if (!(j & 1)) {  // (k, t), |t| <= tk: along b
        const int px = cx + k * ax - tk * bx, py = cy + k * ay - tk * by;
        const int qx = cx + k * ax + tk * bx, qy = cy + k * ay + tk * by;
        if (rect(px, py, qx, qy) > 0) {
          seg_minmax(px, py, bx, by, 2 * tk + 1, mn, mx);
          break;
        }
      } else {  // (u, k), tk < u <= k along a; (k, v), tk < v < k along b
        const int p1x = cx + (tk + 1) * ax + k * bx, p1y = cy + (tk + 1) * ay + k * by;
        const int q1x = cx + k * ax + k * bx, q1y = cy + k * ay + k * by;
        const int n1 = k - tk, n2 = k - 1 - tk;
        const int p2x = cx + k * ax + (tk + 1) * bx, p2y = cy + k * ay + (tk + 1) * by;
        const int q2x = cx + k * ax + (k - 1) * bx, q2y = cy + k * ay + (k - 1) * by;
        const int c1 = rect(p1x, p1y, q1x, q1y);
        const int c2 = n2 > 0 ? rect(p2x, p2y, q2x, q2y) : 0;
        if (c1 + c2 > 0) {
          seg_minmax(p1x, p1y, ax, ay, n1, mn, mx);
          if (n2 > 0) seg_minmax(p2x, p2y, bx, by, n2, mn, mx);
          break;
        }
      }
    }
  }
  // reading B2: max - min > T_neg >= 0 implies two found cells
  out.neg[c] = (mx != INT32_MIN && (int64_t)mx - (int64_t)mn > lp.T_neg) ? 1 : 0;
}

// The same sweep with temporal blocking (TMA lines, 16-byte rows): each
// consumer warp keeps the keys of kS segments of 32 - 2 kNegH apex positions
// in registers, plus kNegH halo lanes on each side, and advances them kNegH
// line steps at a time with shuffles (kNegH = 4 measured best of 4 / 6 / 8) -- no block barrier inside a super-step,
// since an error entering at a segment edge moves one lane per line step and
// never reaches the owned lanes.  Owned keys go through double-buffered shared
// state once per super-step (one named barrier); a ring slot is released when
// every consumer warp has arrived on its `empty` barrier.
#ifndef GVOM_NEG_H
#define GVOM_NEG_H 4
#endif
constexpr int kNegH = GVOM_NEG_H;  // line steps per super-step = halo lanes per side
constexpr int kNegCore = 32 - 2 * kNegH;

template <int kS>
__global__ void __launch_bounds__(1024) k_negative_tb(const Dims d, const LayerParams lp,
                                                      const LayerPtrs out, int T, int R, int W) {
  extern __shared__ __align__(16) uint32_t sm[];
  __shared__ __align__(8) uint64_t full[kNegRing], empty[kNegRing];
  const int cone = blockIdx.y;               // 0:+x 1:-x 2:+y 3:-y
  const bool alongx = cone < 2;              // sweep over x (lines = columns)
  const int dir = (cone & 1) ? -1 : 1;       // ring lines lie at p + dir*k
  const int A = alongx ? d.nx : d.ny;        // lines
  const int K = lp.neg_cells;
  // cross positions held: a line's keys [c0, c1) (rows [row0, row1) of a slab
  // plus a K + 1 halo for the x sweeps; the cells beyond count as outside the
  // map, which cannot reach an emitted cell: its cone spans +-K cross cells)
  const int LB = alongx ? d.ny : d.nx;       // keys per source line
  int c0 = 0, c1 = LB;
  if (alongx) {
    c0 = max(0, (lp.row0 - K - 1) & ~3);
    c1 = min(LB, (lp.row1 + K + 1 + 3) & ~3);
  }
  const int B = c1 - c0;                     // cross positions per line
  const int NB = B + 2 * K + 2;              // apex cross positions -K-1 .. B+K
  const int GL = neg_guard_left(K);
  const int LS = neg_line_stride(B, K);
  const int nthr = W * 32;                   // consumer threads
  const int e0 = alongx ? 0 : lp.row0, e1 = alongx ? d.nx : lp.row1;  // lines emitted
  const uint32_t ONE = 1u << lp.neg_qb;
  const uint32_t NF = (uint32_t)(K + 1) << lp.neg_qb;  // not found
  const uint32_t QM = ONE - 1u;
  uint32_t* ring = sm;                       // [R][2][LS]
  uint32_t* SA = ring + (size_t)R * 2 * LS;  // [2][NB] owned A keys (double buffer)
  uint32_t* SB = SA + 2 * NB;                // [2][NB] owned B keys
  const uint32_t* __restrict__ srcA = (alongx ? out.negAT : out.negA) + c0;
  const uint32_t* __restrict__ srcB = (alongx ? out.negBT : out.negB) + c0;
  const int p0 = e0 + blockIdx.x * T;
  if (p0 >= e1) return;
  const int p1 = min(e1, p0 + T);
  int pstart, nsteps;
  if (dir > 0) {
    pstart = min(A - 1, p1 - 1 + K);
    nsteps = pstart - p0 + 1;
  } else {
    pstart = max(0, p0 - K);
    nsteps = p1 - pstart;
  }
  const uint32_t line_bytes = (uint32_t)B * 4u;
  for (int i = threadIdx.x; i < 2 * NB; i += blockDim.x) {
    SA[i] = NF;
    SB[i] = NF;
  }
  for (int i = threadIdx.x; i < R * 2 * (LS - B); i += blockDim.x) {
    const int line = i / (LS - B), g = i - line * (LS - B);
    ring[(size_t)line * LS + (g < GL ? g : g + B)] = NF;
  }
  if (threadIdx.x == 0) {
    for (int j = 0; j < R; ++j) {
      mbar_init(&full[j], 1);
      mbar_init(&empty[j], (uint32_t)W);  // one arrival per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x >= nthr) {
    // ---------------- producer warp (as in k_negative) ----------------
    if (threadIdx.x == nthr) {
      int j = 0;
      uint32_t ph = 0;
      for (int st = 0; st < nsteps; ++st) {
        if (st >= R) mbar_wait(&empty[j], ph ^ 1u);
        const int pl = pstart - dir * st + dir;
        if (pl >= 0 && pl < A) {
          uint32_t* dst = ring + (size_t)j * 2 * LS + GL;
          const uint32_t b = (uint32_t)__cvta_generic_to_shared(&full[j]);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b),
                       "r"(2u * line_bytes)
                       : "memory");
          tma_copy(dst, srcA + (int64_t)pl * LB, line_bytes, &full[j]);
          tma_copy(dst + LS, srcB + (int64_t)pl * LB, line_bytes, &full[j]);
        } else {
          mbar_arrive(&full[j]);
        }
        if (++j == R) {
          j = 0;
          ph ^= 1u;
        }
      }
    }
    return;
  }
  // ---------------- consumers ----------------
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const bool owner = lane >= kNegH && lane < 32 - kNegH;
  uint32_t a[kS], b[kS];
  int pos[kS];
  bool live[kS];
#pragma unroll
  for (int s = 0; s < kS; ++s) {
    pos[s] = 1 + (warp + s * W) * kNegCore - kNegH + lane;  // apex position of the lane
    live[s] = pos[s] >= 1 && pos[s] <= NB - 2;
  }
  int j = 0, buf = 0;
  uint32_t ph = 0;
  for (int st0 = 0; st0 < nsteps; st0 += kNegH) {
#pragma unroll
    for (int s = 0; s < kS; ++s) {
      a[s] = live[s] ? SA[buf * NB + pos[s]] : NF;
      b[s] = live[s] ? SB[buf * NB + pos[s]] : NF;
    }
    const int st1 = min(nsteps, st0 + kNegH);
    for (int st = st0; st < st1; ++st) {
      const int p = pstart - dir * st;
      const int pl = p + dir;
      const bool inmap = pl >= 0 && pl < A;
      const bool emit = p >= p0 && p < p1;
      mbar_wait(&full[j], ph);
      const uint32_t* ta = ring + (size_t)j * 2 * LS + GL - K - 2;  // apex i: ta[i..i+2]
      const uint32_t* tb = ta + LS;
#pragma unroll
      for (int s = 0; s < kS; ++s) {
        const uint32_t au = __shfl_up_sync(0xffffffffu, a[s], 1);
        const uint32_t ad = __shfl_down_sync(0xffffffffu, a[s], 1);
        const uint32_t bu = __shfl_up_sync(0xffffffffu, b[s], 1);
        const uint32_t bd = __shfl_down_sync(0xffffffffu, b[s], 1);
        uint32_t ka = min(min(au, a[s]), ad) + ONE;
        uint32_t kb = min(min(bu, b[s]), bd) + ONE;
        const int i = pos[s];
        if (inmap && live[s]) {
          ka = min(ka, min(min(ta[i], ta[i + 1]), ta[i + 2]));
          kb = min(kb, min(min(tb[i], tb[i + 1]), tb[i + 2]));
        }
        ka = live[s] ? min(ka, NF) : NF;
        kb = live[s] ? min(kb, NF) : NF;
        a[s] = ka;
        b[s] = kb;
        const int bx = i - K - 1, bg = bx + c0;
        if (emit && owner && ka < NF && (unsigned)bx < (unsigned)B &&
            (!alongx || (bg >= lp.row0 && bg < lp.row1))) {
          const int64_t cell = alongx ? (int64_t)bg * d.nx + p : (int64_t)p * d.nx + bg;
          atomicMin(out.nmin + cell, (int32_t)(ka & QM));
          atomicMax(out.nmax + cell, (int32_t)(QM - (kb & QM)));
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[j]);  // this warp is done with slot j
      if (++j == R) {
        j = 0;
        ph ^= 1u;
      }
    }
    // owned keys to the other state buffer, then one barrier per super-step
#pragma unroll
    for (int s = 0; s < kS; ++s)
      if (owner && live[s]) {
        SA[(buf ^ 1) * NB + pos[s]] = a[s];
        SB[(buf ^ 1) * NB + pos[s]] = b[s];
      }
    asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
    buf ^= 1;
  }
}

// O10 decision from the cone sweeps' min / max: undefined cell and
// max F - min F > T_neg (T_neg >= 0, so this implies |F| >= 2, reading B2);
// rows [row0, row1).  (Folding it into the sweeps' tail -- the block that
// completes a tile pair's four cone counts decides its cells -- measured
// slower: c2 compute_maps 53 vs 45 us.)
__global__ void __launch_bounds__(256) k_neg_decide(const Dims d, const LayerParams lp,
                                                    const LayerPtrs out) {
  const int64_t c = (int64_t)lp.row0 * d.nx + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)lp.row1 * d.nx) return;
  const int32_t mn = __ldg(out.nmin + c), mx = __ldg(out.nmax + c);
  out.neg[c] = (__ldg(out.qs + c) == kQsUndef && mx != INT32_MIN &&
                (int64_t)mx - (int64_t)mn > lp.T_neg)
                   ? 1
                   : 0;
}

// Costmap: weighted per-pixel sum of the layers,
// f32 RN in the order hard, soft, density, negative, slope, roughness,
// unknown; an undefined (NaN) layer contributes 0 (reading B5).
__device__ __forceinline__ float cost_of(const CostWeights& cw, float h, float de, uint8_t hd,
                                         uint8_t so, uint8_t ng, float sl, float ro) {
  float acc = 0.0f;
  acc = __fadd_rn(acc, __fmul_rn(cw.w[0], (float)hd));
  acc = __fadd_rn(acc, __fmul_rn(cw.w[1], (float)so));
  acc = __fadd_rn(acc, __fmul_rn(cw.w[2], isnan(de) ? 0.0f : de));
  acc = __fadd_rn(acc, __fmul_rn(cw.w[3], (float)ng));
  acc = __fadd_rn(acc, __fmul_rn(cw.w[4], isnan(sl) ? 0.0f : sl));
  acc = __fadd_rn(acc, __fmul_rn(cw.w[5], isnan(ro) ? 0.0f : ro));
  acc = __fadd_rn(acc, __fmul_rn(cw.w[6], (isnan(h) && !ng) ? 1.0f : 0.0f));
  return acc;
}

__global__ void __launch_bounds__(256) k_costmap(const Dims d, const LayerPtrs in,
                                                 const CostWeights cw, float* __restrict__ out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)d.nx * d.ny) return;
  out[c] = cost_of(cw, __ldg(in.height + c), __ldg(in.density + c), __ldg(in.hard + c),
                   __ldg(in.soft + c), __ldg(in.neg + c), __ldg(in.slope + c),
                   __ldg(in.rough + c));
}

// Export fused with the costmap (NEXT-4 "fused into export"): each layer
// cell is read once, written to its destination and folded into the cost.
// Destinations in GVOM_LAYER order.
__global__ void __launch_bounds__(256) k_export_cost(const Dims d, const LayerPtrs in,
                                                     const __grid_constant__ CopyJob job,
                                                     const CostWeights cw,
                                                     float* __restrict__ cost) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)d.nx * d.ny) return;
  const float h = __ldcs(in.height + c), de = __ldcs(in.density + c);
  const uint8_t hd = __ldcs(in.hard + c), so = __ldcs(in.soft + c), ng = __ldcs(in.neg + c);
  const float sl = __ldcs(in.slope + c), ro = __ldcs(in.rough + c), sp = __ldcs(in.spread + c);
  static_cast<float*>(job.dst[GVOM_LAYER_HEIGHT])[c] = h;
  static_cast<float*>(job.dst[GVOM_LAYER_DENSITY])[c] = de;
  static_cast<uint8_t*>(job.dst[GVOM_LAYER_HARD])[c] = hd;
  static_cast<uint8_t*>(job.dst[GVOM_LAYER_SOFT])[c] = so;
  static_cast<uint8_t*>(job.dst[GVOM_LAYER_NEGATIVE])[c] = ng;
  static_cast<float*>(job.dst[GVOM_LAYER_SLOPE])[c] = sl;
  static_cast<float*>(job.dst[GVOM_LAYER_ROUGHNESS])[c] = ro;
  static_cast<float*>(job.dst[GVOM_LAYER_SPREAD])[c] = sp;
  cost[c] = cost_of(cw, h, de, hd, so, ng, sl, ro);
}

// merged occupancy bits of the combined map (export path)
__global__ void __launch_bounds__(128) k_merge_bits(const SlotSet ss, const Dims d,
                                                    uint32_t* __restrict__ mbits) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)d.nx * d.ny) return;
  const int x = (int)(c % d.nx), y = (int)(c / d.nx);
  const int64_t outbase = (int64_t)d.nz * c;
  for (int z0 = 0; z0 < d.nz; z0 += 32) {
    uint32_t m = 0;
    for (int k = 0; k < ss.K; ++k) {
      const SlotView& s = ss.s[k];
      const int sx = x + s.dx, sy = y + s.dy;
      if ((unsigned)sx >= (unsigned)d.nx || (unsigned)sy >= (unsigned)d.ny) continue;
      const int64_t cb = (int64_t)d.nz * ((int64_t)sx + (int64_t)d.nx * sy);
      m |= col_bits32(s.bits, d.W, cb, z0 + s.dz, d.nz);
    }
    if (!m) continue;
    const int64_t p = outbase + z0;
    const int sh = (int)(p & 31);
    atomicOr(mbits + (p >> 5), m << sh);
    if (sh) {
      const uint32_t hi = m >> (32 - sh);
      if (hi) atomicOr(mbits + (p >> 5) + 1, hi);
    }
  }
}

__global__ void __launch_bounds__(256) k_merge_write(const SlotSet ss, const Dims d,
                                                     const uint32_t* __restrict__ mbits,
                                                     const uint32_t* __restrict__ mprefix,
                                                     int32_t* __restrict__ lut,
                                                     gvom_voxel* __restrict__ data) {
  const int64_t L = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (L >= d.V) return;
  const int z = (int)(L % d.nz);
  const int64_t col = L / d.nz;
  const int x = (int)(col % d.nx), y = (int)(col / d.nx);
  uint64_t H = 0, Mi = 0, M1 = 0, M2 = 0;
  uint32_t mn = 0xffffffffu;
  for (int k = 0; k < ss.K; ++k) {
    const SlotView& s = ss.s[k];
    const int ux = x + s.dx, uy = y + s.dy, uz = z + s.dz;
    if ((unsigned)ux >= (unsigned)d.nx || (unsigned)uy >= (unsigned)d.ny ||
        (unsigned)uz >= (unsigned)d.nz)
      continue;
    const int64_t Ls = (int64_t)uz + (int64_t)d.nz * ((int64_t)ux + (int64_t)d.nx * uy);
    uint32_t r;
    if (slot_rank(s, Ls, r)) {
      const gvom_voxel v = s.data[r];
      H += v.hits;
      Mi += v.misses;
      mn = min(mn, v.min_dz);
      M1 += v.m1;
      M2 += v.m2;
    } else {
      Mi += (uint64_t)(-1ll - (int64_t)__ldg(s.lut + Ls));
    }
  }
  const uint32_t bw = __ldg(mbits + (L >> 5));
  const int bit = (int)(L & 31);
  if ((bw >> bit) & 1u) {
    const uint32_t rank = __ldg(mprefix + (L >> 5)) + __popc(bw & ((1u << bit) - 1u));
    lut[L] = (int32_t)rank;
    gvom_voxel v;
    v.hits = (uint32_t)H;
    v.misses = (uint32_t)Mi;
    v.min_dz = mn;
    v.reserved = 0;
    v.m1 = M1;
    v.m2 = M2;
    data[rank] = v;
  } else {
    const uint64_t nm = Mi < kMissSat ? Mi : kMissSat;
    lut[L] = -1 - (int32_t)nm;
  }
}

// All 2D layers in one launch: blockIdx.y selects the layer; 16-byte chunks.
__device__ __forceinline__ uint32_t neg_decision(const NegDecide& dec, int32_t q, int32_t mn,
                                                 int32_t mx) {
  return (q == kQsUndef && mx != INT32_MIN && (int64_t)mx - (int64_t)mn > dec.T_neg) ? 1u : 0u;
}

__global__ void __launch_bounds__(256) k_export_layers(const __grid_constant__ CopyJob job,
                                                       const __grid_constant__ NegDecide dec) {
  const int l = blockIdx.y;
  if (dec.on && l == GVOM_LAYER_NEGATIVE) {
    // k_neg_decide's rule on the way out: four cells per thread, 16-byte loads
    // of q_s / nmin / nmax, one 4-byte store to the caller and to the layer
    const int64_t n = job.bytes[l], n4 = n >> 2;
    const int4* q4 = reinterpret_cast<const int4*>(dec.qs);
    const int4* a4 = reinterpret_cast<const int4*>(dec.nmin);
    const int4* b4 = reinterpret_cast<const int4*>(dec.nmax);
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x) {
      const int4 q = __ldcs(q4 + i), a = __ldcs(a4 + i), b = __ldcs(b4 + i);
      const uint32_t v = neg_decision(dec, q.x, a.x, b.x) | neg_decision(dec, q.y, a.y, b.y) << 8 |
                         neg_decision(dec, q.z, a.z, b.z) << 16 |
                         neg_decision(dec, q.w, a.w, b.w) << 24;
      reinterpret_cast<uint32_t*>(job.dst[l])[i] = v;
      reinterpret_cast<uint32_t*>(dec.neg)[i] = v;
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
      const int64_t c = (n4 << 2) + threadIdx.x;
      const uint8_t v = (uint8_t)neg_decision(dec, dec.qs[c], dec.nmin[c], dec.nmax[c]);
      reinterpret_cast<uint8_t*>(job.dst[l])[c] = v;
      dec.neg[c] = v;
    }
    return;
  }
  const int64_t n16 = job.bytes[l] >> 4;
  const uint4* __restrict__ src = reinterpret_cast<const uint4*>(job.src[l]);
  uint4* __restrict__ dst = reinterpret_cast<uint4*>(job.dst[l]);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n16;
       i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = __ldcs(src + i);
  if (blockIdx.x == 0 && threadIdx.x < (job.bytes[l] & 15)) {
    const int64_t b = (n16 << 4) + threadIdx.x;
    reinterpret_cast<uint8_t*>(job.dst[l])[b] = reinterpret_cast<const uint8_t*>(job.src[l])[b];
  }
}

inline unsigned cells_blocks(const Dims& d, int tpb) {
  return (unsigned)(((int64_t)d.nx * d.ny + tpb - 1) / tpb);
}

}  // namespace

cudaError_t launch_columns(const SlotSet& ss, const Dims& d, const LayerParams& lp,
                           const LayerPtrs& out, cudaStream_t st, int64_t cbeg, int64_t cend) {
  if (cend < 0) cend = (int64_t)d.nx * d.ny;
  if (cend <= cbeg) return cudaSuccess;
  const int64_t lanes = (cend - cbeg) << ss.kp_log2;
  // GVOM_COL_FAST=1: the three-round-trip kernel when the band fits the 64-z
  // window (A/B; 62 registers, measured slower on c2/c3 -- columns 33.2 vs
  // 27.1 us -- and a tie on c4, so off by default)
  static int fast = -1;
  if (fast < 0) {
    const char* e = getenv("GVOM_COL_FAST");
    fast = e && atoi(e) == 1 ? 1 : 0;
  }
  const int64_t nb = (65535 + lp.T_hi) >> 16;
  if (fast && nb < 32) {
    k_columns_fast<<<(unsigned)((lanes + 255) / 256), 256, 0, st>>>(ss, d, lp, out, cbeg, cend,
                                                                     (int)nb);
    return cudaGetLastError();
  }
  // GVOM_COL_EARLY=1: the edge voxels' loads issued before the band's (A/B:
  // 59 instead of 48 registers, measured slower -- c2 columns 31.1 vs 27.1 us)
  static int early = -1;
  if (early < 0) {
    const char* e = getenv("GVOM_COL_EARLY");
    early = e && atoi(e) == 1 ? 1 : 0;
  }
  if (early)
    k_columns<true><<<(unsigned)((lanes + 255) / 256), 256, 0, st>>>(ss, d, lp, out, cbeg, cend);
  else
    k_columns<false><<<(unsigned)((lanes + 255) / 256), 256, 0, st>>>(ss, d, lp, out, cbeg, cend);
  return cudaGetLastError();
}

cudaError_t launch_slope(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                         cudaStream_t st) {
  static int old_kernel = -1;  // GVOM_SLOPE_COMPACT=1: the compacted kernel (A/B)
  if (old_kernel < 0) {
    const char* e = getenv("GVOM_SLOPE_COMPACT");
    old_kernel = e && atoi(e) ? 0 : 1;
  }
  if (old_kernel) {
    const int rows = lp.row1 - lp.row0;
    const dim3 grid((d.nx + kSlopeTX - 1) / kSlopeTX, (rows + kSlopeTY - 1) / kSlopeTY);
    k_slope<<<grid, dim3(kSlopeTX, kSlopeTY), 0, st>>>(d, lp, out);
  } else {
    const int rows = lp.row1 - lp.row0;
    const dim3 grid((d.nx + kSlope2TX - 1) / kSlope2TX, (rows + kSlope2TY - 1) / kSlope2TY);
    k_slope_c<<<grid, kSlope2Threads, 0, st>>>(d, lp, out);
  }
  return cudaGetLastError();
}

#ifndef GVOM_NEG_TB
#define GVOM_NEG_TB 1
#endif
inline bool neg_tb_enabled() { return GVOM_NEG_TB != 0; }  // A/B knob

cudaError_t launch_negative(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                            cudaStream_t st, bool decide) {
  const int A = d.nx > d.ny ? d.nx : d.ny, B = A;  // smem sized for the longest line
  const int K = lp.neg_cells;
  // tiles: about one block per SM over the emitted lines of the 4 cones (rows
  // [row0, row1) for the y sweeps, every column for the x sweeps), >= 8 lines
  const int rows = lp.row1 - lp.row0;
  int T = (2 * d.nx + 2 * rows + d.sms - 1) / d.sms;
  T = T < 8 ? 8 : ((T + 7) / 8) * 8;
  {  // GVOM_NEG_T: lines per tile (A/B)
    static int t_env = -1;
    if (t_env < 0) {
      const char* e = getenv("GVOM_NEG_T");
      t_env = e ? atoi(e) : 0;
    }
    if (t_env >= 2) T = t_env;
  }
  const size_t NB = (size_t)B + 2 * (size_t)K + 2;
  const size_t slot = neg_slot_bytes(B, K), state = neg_state_bytes(B, K);
  // ring depth: as many slots as shared memory allows, up to kNegRing
  // (gvom_create guarantees at least 2, neg_sweep_fits)
  if (!neg_sweep_fits(B, K)) return cudaErrorInvalidConfiguration;
  int R = (int)((kNegSmemMax - state) / slot);
  R = R > kNegRing ? kNegRing : R;
  {  // GVOM_NEG_RMAX: cap the ring depth (A/B: leaves shared memory for the
     // plane-fit blocks that run concurrently on the main stream)
    static int rmax = -1;
    if (rmax < 0) {
      const char* e = getenv("GVOM_NEG_RMAX");
      rmax = e ? atoi(e) : 0;
    }
    if (rmax >= 2 && R > rmax) R = rmax;
  }
  const size_t smem = state + (size_t)R * slot;
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(
        k_negative, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  const int lines = d.nx > rows ? d.nx : rows;
  const dim3 grid((unsigned)((lines + T - 1) / T), 4);
  // temporally blocked sweep when the rows of both sweep directions are whole
  // 16-byte chunks (TMA) and up to 4 segments per warp (31 warps) cover a
  // line: c2 18.3 -> 15.1 us, c4 29.4 -> 27.0 us, c5 (2 segments) 110 -> 97 us
  const int nseg = (int)((NB - 2 + kNegCore - 1) / kNegCore);
#ifndef GVOM_NEG_TB_MAXS
#define GVOM_NEG_TB_MAXS 4  // segments per warp (A/B knob)
#endif
  const int W = nseg < 31 ? nseg : 31;
  const int S = (nseg + W - 1) / W;
  if ((d.nx & 3) == 0 && (d.ny & 3) == 0 && S <= GVOM_NEG_TB_MAXS && neg_tb_enabled()) {
    auto kern = S == 1 ? k_negative_tb<1> : S == 2 ? k_negative_tb<2> : k_negative_tb<4>;
    if (smem > 48 * 1024) {
      const cudaError_t e =
          cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    kern<<<grid, W * 32 + 32, smem, st>>>(d, lp, out, T, R, W);
  } else {
    // consumers: one apex position each per pass (up to 992), + 1 producer warp
    int nthr = (int)((NB - 2 + 31) / 32) * 32;
    if (nthr > 1024 - 32) nthr = 1024 - 32;
    k_negative<<<grid, nthr + 32, smem, st>>>(d, lp, out, T, R);
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess || !decide) return e;
  return launch_neg_decide(d, lp, out, st);
}

cudaError_t launch_negative8(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                             cudaStream_t st) {
  // 32 x 32 tiles (1024 threads) when they give at least two blocks per SM,
  // else 16 x 16 (more blocks for small maps, more halo per cell)
  const int64_t t32 = ((d.nx + 31) / 32) * (int64_t)((d.ny + 31) / 32);
  const int tile = t32 >= 2 * (int64_t)d.sms ? 32 : 16;
  const size_t smem = neg8_smem_bytes(lp.neg_cells, tile);
  if (smem > kNegSmemMax) return cudaErrorInvalidConfiguration;
  const dim3 grid((unsigned)((d.nx + tile - 1) / tile), (unsigned)((d.ny + tile - 1) / tile));
  if (tile == 32) {
    if (smem > 48 * 1024) {
      const cudaError_t e = cudaFuncSetAttribute(
          k_negative8<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    k_negative8<32><<<grid, 1024, smem, st>>>(d, lp, out);
  } else {
    if (smem > 48 * 1024) {
      const cudaError_t e = cudaFuncSetAttribute(
          k_negative8<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
    }
    k_negative8<16><<<grid, 256, smem, st>>>(d, lp, out);
  }
  return cudaGetLastError();
}

cudaError_t launch_export_layers(const CopyJob& job, cudaStream_t st, const NegDecide& dec) {
  int64_t mx = 0;
  for (int l = 0; l < GVOM_LAYER_COUNT; ++l) mx = job.bytes[l] > mx ? job.bytes[l] : mx;
  int64_t blocks = ((mx >> 4) + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 4) blocks = 148 * 4;
  k_export_layers<<<dim3((unsigned)blocks, GVOM_LAYER_COUNT), 256, 0, st>>>(job, dec);
  return cudaGetLastError();
}

cudaError_t launch_neg_decide(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                              cudaStream_t st) {
  const int64_t dc = (int64_t)(lp.row1 - lp.row0) * d.nx;
  if (dc <= 0) return cudaSuccess;
  k_neg_decide<<<(unsigned)((dc + 255) / 256), 256, 0, st>>>(d, lp, out);
  return cudaGetLastError();
}

cudaError_t launch_costmap(const Dims& d, const LayerPtrs& in, const CostWeights& cw, float* out,
                           cudaStream_t st) {
  k_costmap<<<cells_blocks(d, 256), 256, 0, st>>>(d, in, cw, out);
  return cudaGetLastError();
}

cudaError_t launch_export_cost(const Dims& d, const LayerPtrs& in, const CopyJob& job,
                               const CostWeights& cw, float* cost, cudaStream_t st) {
  k_export_cost<<<cells_blocks(d, 256), 256, 0, st>>>(d, in, job, cw, cost);
  return cudaGetLastError();
}

cudaError_t launch_merge_bits(const SlotSet& ss, const Dims& d, uint32_t* mbits, cudaStream_t st) {
  k_merge_bits<<<cells_blocks(d, 128), 128, 0, st>>>(ss, d, mbits);
  return cudaGetLastError();
}

cudaError_t launch_merge_write(const SlotSet& ss, const Dims& d, const uint32_t* mbits,
                               const uint32_t* mprefix, int32_t* lut, gvom_voxel* data,
                               cudaStream_t st) {
  const int64_t blocks = (d.V + 255) / 256;
  k_merge_write<<<(unsigned)blocks, 256, 0, st>>>(ss, d, mbits, mprefix, lut, data);
  return cudaGetLastError();
}

}  // namespace gvom
