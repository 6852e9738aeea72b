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

struct Merged {
  uint64_t H, Mi;
  uint32_t mn;
};

// O7 for one output voxel (x, y, z): sum hits/misses, min of min_dz.
__device__ __forceinline__ Merged merge_voxel(const SlotSet& ss, const Dims& d, int x, int y,
                                              int z) {
  Merged m{0, 0, 0xffffffffu};
  for (int k = 0; k < ss.K; ++k) {
    const SlotView& s = ss.s[k];
    const int ux = x + s.dx, uy = y + s.dy, uz = z + s.dz;
    if ((unsigned)ux >= (unsigned)d.nx || (unsigned)uy >= (unsigned)d.ny ||
        (unsigned)uz >= (unsigned)d.nz)
      continue;
    const int64_t L = (int64_t)uz + (int64_t)d.nz * ((int64_t)ux + (int64_t)d.nx * uy);
    uint32_t r;
    if (slot_rank(s, L, r)) {
      const uint4 row = __ldg(reinterpret_cast<const uint4*>(s.data + r));
      m.H += row.x;
      m.Mi += row.y;
      m.mn = min(m.mn, row.z);
    } else {
      m.Mi += (uint64_t)(-1ll - (int64_t)__ldg(s.lut + L));
    }
  }
  return m;
}

__global__ void __launch_bounds__(128) k_columns(const SlotSet ss, const Dims d,
                                                 const LayerParams lp, const LayerPtrs out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)d.nx * d.ny) return;
  const int x = (int)(c % d.nx), y = (int)(c / d.nx);
  // z*: lowest z occupied in any buffer map (O8)
  int zs = -1;
  for (int z0 = 0; z0 < d.nz && zs < 0; z0 += 32) {
    uint32_t m = 0;
    for (int k = 0; k < ss.K; ++k) {
      const SlotView& s = ss.s[k];
      const int sx = x + s.dx, sy = y + s.dy;
      if ((unsigned)sx >= (unsigned)d.nx || (unsigned)sy >= (unsigned)d.ny) continue;
      const int64_t cb = (int64_t)d.nz * ((int64_t)sx + (int64_t)d.nx * sy);
      m |= col_bits32(s.bits, d.W, cb, z0 + s.dz, d.nz);
    }
    if (m) zs = z0 + __ffs(m) - 1;
  }
  out.hard[c] = 0;
  out.soft[c] = 0;
  if (zs < 0) {
    out.height[c] = __int_as_float(0x7fc00000);
    out.density[c] = __int_as_float(0x7fc00000);
    out.qs[c] = kQsUndef;
    return;
  }
  const Merged ms = merge_voxel(ss, d, x, y, zs);
  const int64_t q_s = 65536ll * zs + (int64_t)ms.mn;
  out.qs[c] = (int32_t)q_s;
  out.height[c] = (float)(((double)(lp.o_z * 65536 + q_s) * lp.res) / 65536.0);
  // obstacle band: occupied z with T_lo <= 65536 z + mn(z) - q_s <= T_hi (A18)
  const int64_t zhi64 = (lp.T_hi + q_s) >> 16;
  const int zhi = (int)(zhi64 < (int64_t)d.nz - 1 ? zhi64 : (int64_t)d.nz - 1);
  uint64_t SH = 0, SW = 0;
  for (int z0 = zs & ~31; z0 <= zhi; z0 += 32) {
    uint32_t m = 0;
    for (int k = 0; k < ss.K; ++k) {
      const SlotView& s = ss.s[k];
      const int sx = x + s.dx, sy = y + s.dy;
      if ((unsigned)sx >= (unsigned)d.nx || (unsigned)sy >= (unsigned)d.ny) continue;
      const int64_t cb = (int64_t)d.nz * ((int64_t)sx + (int64_t)d.nx * sy);
      m |= col_bits32(s.bits, d.W, cb, z0 + s.dz, d.nz);
    }
    // keep z in (zs, zhi]: the surface voxel itself has dq = mn(zs) - mn(zs) = 0
    // which is in the band only if T_lo <= 0; handle it explicitly below.
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      const int z = z0 + b;
      if (z < zs || z > zhi) continue;
      const Merged mz = (z == zs) ? ms : merge_voxel(ss, d, x, y, z);
      const int64_t dq = (65536ll * z + (int64_t)mz.mn) - q_s;
      if (dq >= lp.T_lo && dq <= lp.T_hi) {
        SH += mz.H;
        SW += mz.H + mz.Mi;
      }
    }
  }
  if (SH == 0) {
    out.density[c] = 0.0f;
    return;
  }
  out.density[c] = (float)((double)SH / (double)SW);
  if (65536ull * SH >= (uint64_t)lp.tau * SW)
    out.hard[c] = 1;
  else
    out.soft[c] = 1;
}

__device__ __forceinline__ int64_t det3(int64_t a, int64_t b, int64_t c, int64_t d, int64_t e,
                                        int64_t f, int64_t g, int64_t h, int64_t i) {
  return a * (e * i - f * h) - b * (d * i - f * g) + c * (d * h - e * g);
}

// O9: plane fit over the defined in-map cells of the N x N window
__global__ void __launch_bounds__(128) k_slope(const Dims d, const LayerParams lp,
                                               const LayerPtrs out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)d.nx * d.ny) return;
  const int x = (int)(c % d.nx), y = (int)(c / d.nx);
  const float qnan = __int_as_float(0x7fc00000);
  const int32_t* __restrict__ qs = out.qs;
  const int32_t qc = __ldg(qs + c);
  if (qc == kQsUndef) {
    out.slope[c] = qnan;
    out.rough[c] = qnan;
    return;
  }
  const int r = (lp.slope_window - 1) / 2;
  int64_t n = 0, Su = 0, Sv = 0, Suu = 0, Svv = 0, Suv = 0, Sz = 0, Suz = 0, Svz = 0;
  for (int v = -r; v <= r; ++v) {
    const int yy = y + v;
    if ((unsigned)yy >= (unsigned)d.ny) continue;
    for (int u = -r; u <= r; ++u) {
      const int xx = x + u;
      if ((unsigned)xx >= (unsigned)d.nx) continue;
      const int32_t q = __ldg(qs + xx + (int64_t)d.nx * yy);
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
  for (int v = -r; v <= r; ++v) {
    const int yy = y + v;
    if ((unsigned)yy >= (unsigned)d.ny) continue;
    for (int u = -r; u <= r; ++u) {
      const int xx = x + u;
      if ((unsigned)xx >= (unsigned)d.nx) continue;
      const int32_t q = __ldg(qs + xx + (int64_t)d.nx * yy);
      if (q == kQsUndef) continue;
      const int64_t z = (int64_t)q - qc;
      const double e = (double)(det * z - Da * u - Db * v - Dc);
      acc += e * e;
    }
  }
  const double sc = lp.res / 65536.0;
  out.rough[c] = (float)(acc / ((double)det * (double)det * (double)n) * (sc * sc));
}

// O10: negative obstacles for undefined cells
__global__ void __launch_bounds__(128) k_negative(const Dims d, const LayerParams lp,
                                                  const LayerPtrs out) {
  const int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= (int64_t)d.nx * d.ny) return;
  const int x = (int)(c % d.nx), y = (int)(c / d.nx);
  const int32_t* __restrict__ qs = out.qs;
  if (__ldg(qs + c) != kQsUndef) {
    out.neg[c] = 0;
    return;
  }
  int64_t fmin = INT64_MAX, fmax = INT64_MIN, fcount = 0;
  for (int cone = 0; cone < 4; ++cone) {
    for (int k = 1; k <= lp.neg_cells; ++k) {
      bool found = false;
      for (int t = -k; t <= k; ++t) {
        int xx, yy;
        if (cone == 0) {
          xx = x + k;
          yy = y + t;
        } else if (cone == 1) {
          xx = x - k;
          yy = y + t;
        } else if (cone == 2) {
          xx = x + t;
          yy = y + k;
        } else {
          xx = x + t;
          yy = y - k;
        }
        if ((unsigned)xx >= (unsigned)d.nx || (unsigned)yy >= (unsigned)d.ny) continue;
        const int32_t q = __ldg(qs + xx + (int64_t)d.nx * yy);
        if (q == kQsUndef) continue;
        found = true;
        fmin = min(fmin, (int64_t)q);
        fmax = max(fmax, (int64_t)q);
        ++fcount;
      }
      if (found) break;
    }
  }
  out.neg[c] = (fcount >= 2 && (fmax - fmin) > lp.T_neg) ? 1 : 0;
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

inline unsigned cells_blocks(const Dims& d, int tpb) {
  return (unsigned)(((int64_t)d.nx * d.ny + tpb - 1) / tpb);
}

}  // namespace

cudaError_t launch_columns(const SlotSet& ss, const Dims& d, const LayerParams& lp,
                           const LayerPtrs& out, cudaStream_t st) {
  k_columns<<<cells_blocks(d, 128), 128, 0, st>>>(ss, d, lp, out);
  return cudaGetLastError();
}

cudaError_t launch_slope(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                         cudaStream_t st) {
  k_slope<<<cells_blocks(d, 128), 128, 0, st>>>(d, lp, out);
  return cudaGetLastError();
}

cudaError_t launch_negative(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                            cudaStream_t st) {
  k_negative<<<cells_blocks(d, 128), 128, 0, st>>>(d, lp, out);
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
