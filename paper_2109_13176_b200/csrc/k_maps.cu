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

// O7 + O8 fused, one warp per output column.  Lane (g, k): slot k = lane mod
// 2^lg of group g = lane >> lg.  Groups scan different 32-z chunks, then
// evaluate different candidate voxels of the column in parallel; each voxel is
// the sum / min over the slots of its group (segmented shuffles).
__global__ void __launch_bounds__(256) k_columns(const __grid_constant__ SlotSet ss, const Dims d,
                                                 const LayerParams lp, const LayerPtrs out) {
  const int lane = threadIdx.x & 31;
  const int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (c >= (int64_t)d.nx * d.ny) return;  // warp-uniform
  const int x = (int)(c % d.nx), y = (int)(c / d.nx);
  const int lg = ss.kp_log2;
  const int k = lane & ((1 << lg) - 1);
  const int g = lane >> lg;
  const int G = 32 >> lg;
  // this lane's slot column
  bool col = false;
  int64_t cb = 0;
  int dz = 0;
  const uint32_t* bits = nullptr;
  const uint32_t* wpre = nullptr;
  const gvom_voxel* data = nullptr;
  const int32_t* lut = nullptr;
  if (k < ss.K) {
    const SlotView& s = ss.s[k];
    const int sx = x + s.dx, sy = y + s.dy;
    if ((unsigned)sx < (unsigned)d.nx && (unsigned)sy < (unsigned)d.ny) {
      col = true;
      cb = (int64_t)d.nz * ((int64_t)sx + (int64_t)d.nx * sy);
      dz = s.dz;
      bits = s.bits;
      wpre = s.wprefix;
      data = s.data;
      lut = s.lut;
    }
  }
  // ---- z*: lowest z occupied in any buffer map ----
  int zs = -1;
  for (int zb = 0; zb < d.nz && zs < 0; zb += 32 * G) {
    const int z0 = zb + 32 * g;
    uint32_t m = (col && z0 < d.nz) ? col_bits32(bits, d.W, cb, z0 + dz, d.nz) : 0u;
    m = grp_or(m, lg);
    const unsigned nzg = __ballot_sync(0xffffffffu, m != 0u && k == 0);
    if (nzg) {
      const int gl = __ffs(nzg) - 1;  // leader lane of the lowest non-empty chunk
      const uint32_t mm = __shfl_sync(0xffffffffu, m, gl);
      zs = zb + 32 * (gl >> lg) + __ffs(mm) - 1;
    }
  }
  if (zs < 0) {
    if (lane == 0) {
      out.hard[c] = 0;
      out.soft[c] = 0;
      out.height[c] = __int_as_float(0x7fc00000);
      out.density[c] = __int_as_float(0x7fc00000);
      out.qs[c] = kQsUndef;
    }
    return;
  }
  // ---- candidates: merged occupancy in a window starting at z* ----
  const int span = (int)((lp.T_hi >> 16) + 1);  // band top is at most z* + span
  int64_t q_s = 0;
  int zhi = zs;
  uint64_t SH = 0, SW = 0;
  bool have_qs = false;
  for (int w0 = zs; w0 <= zs + span && w0 < d.nz; w0 += 32) {
    uint32_t wm = col ? col_bits32(bits, d.W, cb, w0 + dz, d.nz) : 0u;
    wm = grp_or(wm, lg);  // identical in every group
    if (have_qs) {
      const int lim = zhi - w0;  // keep z <= zhi
      if (lim < 0) break;
      if (lim < 31) wm &= (2u << lim) - 1u;
    }
    while (wm) {
      // group g takes the g-th remaining candidate of this batch
      uint32_t t = wm;
      for (int i = 0; i < g && t; ++i) t &= t - 1;
      const bool has = t != 0u;
      const int z = has ? w0 + __ffs(t) - 1 : -1;
      // remove G candidates from wm
      for (int i = 0; i < G && wm; ++i) wm &= wm - 1;
      uint32_t h = 0, mi = 0, mn = 0xffffffffu;
      if (has && col) {
        const int uz = z + dz;
        if ((unsigned)uz < (unsigned)d.nz) {
          const int64_t L = cb + uz;
          const int64_t wi = L >> 5;
          const int bit = (int)(L & 31);
          const uint32_t bw = __ldg(bits + wi);
          if ((bw >> bit) & 1u) {
            const uint32_t r = __ldg(wpre + wi) + __popc(bw & ((1u << bit) - 1u));
            const uint4 row = __ldg(reinterpret_cast<const uint4*>(data + r));
            h = row.x;
            mi = row.y;
            mn = row.z;
          } else {
            mi = (uint32_t)(-1 - __ldg(lut + L));
          }
        }
      }
      const uint64_t H = grp_add64(h, lg);
      const uint64_t Mi = grp_add64(mi, lg);
      const uint32_t MN = grp_min(mn, lg);
      if (!have_qs) {
        // the first candidate of the first batch (group 0) is z* itself
        const uint32_t mn0 = __shfl_sync(0xffffffffu, MN, 0);
        q_s = 65536ll * zs + (int64_t)mn0;
        const int64_t zh = (lp.T_hi + q_s) >> 16;
        zhi = (int)(zh < (int64_t)d.nz - 1 ? zh : (int64_t)d.nz - 1);
        have_qs = true;
      }
      if (k == 0 && has && z <= zhi) {
        const int64_t dq = (65536ll * z + (int64_t)MN) - q_s;
        if (dq >= lp.T_lo && dq <= lp.T_hi) {
          SH += H;
          SW += H + Mi;
        }
      }
      // drop candidates above zhi (uniform: zhi and wm are warp-uniform)
      const int lim = zhi - w0;
      if (lim < 0)
        wm = 0u;
      else if (lim < 31)
        wm &= (2u << lim) - 1u;
    }
    // (uniform) stop once past zhi
    if (w0 + 32 > zhi) break;
  }
  // sum the group leaders' partial band sums (non-leaders hold 0)
  for (int o = 16; o > 0; o >>= 1) {
    SH += __shfl_xor_sync(0xffffffffu, SH, o);
    SW += __shfl_xor_sync(0xffffffffu, SW, o);
  }
  if (lane == 0) {
    out.qs[c] = (int32_t)q_s;
    out.height[c] = (float)(((double)(lp.o_z * 65536 + q_s) * lp.res) / 65536.0);
    uint8_t hard = 0, soft = 0;
    if (SH == 0) {
      out.density[c] = 0.0f;
    } else {
      out.density[c] = (float)((double)SH / (double)SW);
      if (65536ull * SH >= (uint64_t)lp.tau * SW)
        hard = 1;
      else
        soft = 1;
    }
    out.hard[c] = hard;
    out.soft[c] = soft;
    const int WX = (d.nx + 31) >> 5, WY = (d.ny + 31) >> 5;
    atomicOr(out.rowbits + (int64_t)y * WX + (x >> 5), 1u << (x & 31));
    atomicOr(out.colbits + (int64_t)x * WY + (y >> 5), 1u << (y & 31));
  }
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

// Defined cells of one ring line (a row or column segment [lo, hi]) from the
// defined-surface bitmask; for each, fold q into (min, max, count).
__device__ __forceinline__ bool ring_line(const uint32_t* __restrict__ bm, int lo, int hi,
                                          const int32_t* __restrict__ qs, int64_t q0,
                                          int64_t qstride, int64_t& fmin, int64_t& fmax,
                                          int64_t& fcount) {
  bool found = false;
  for (int wi = lo >> 5; wi <= (hi >> 5); ++wi) {
    uint32_t w = __ldg(bm + wi);
    const int b0 = wi << 5;
    if (lo > b0) w &= ~0u << (lo - b0);
    if (hi < b0 + 31) w &= (2u << (hi - b0)) - 1u;
    while (w) {
      const int i = b0 + __ffs(w) - 1;
      w &= w - 1;
      const int64_t q = __ldg(qs + q0 + qstride * i);
      fmin = min(fmin, q);
      fmax = max(fmax, q);
      ++fcount;
      found = true;
    }
  }
  return found;
}

// O10: negative obstacles for undefined cells.  A block is 32
// consecutive cells x 4 cones: warp w searches cone w for its 32 cells (lanes
// of a warp probe neighbouring rings, so they run similar distances); the
// four cones are combined through shared memory.  Ring k of cone +x is the
// column segment (x+k, y-k..y+k), tested 32 cells per bitmask word.
__global__ void __launch_bounds__(128) k_negative(const Dims d, const LayerParams lp,
                                                  const LayerPtrs out) {
  __shared__ int32_t smin[4][32], smax[4][32], scnt[4][32];
  const int tx = threadIdx.x, cone = threadIdx.y;
  const int64_t cells = (int64_t)d.nx * d.ny;
  const int64_t c = (int64_t)blockIdx.x * 32 + tx;
  const int32_t* __restrict__ qs = out.qs;
  const bool undef = c < cells && __ldg(qs + c) == kQsUndef;
  int64_t fmin = INT64_MAX, fmax = INT64_MIN, fcount = 0;
  if (undef) {
    const int x = (int)(c % d.nx), y = (int)(c / d.nx);
    const int WX = (d.nx + 31) >> 5, WY = (d.ny + 31) >> 5;
    const bool alongx = cone < 2;  // +x / -x cones: ring lines are columns
    const int sgn = (cone & 1) ? -1 : 1;
    const int base = alongx ? x : y;
    const int nline = alongx ? d.nx : d.ny;
    const int center = alongx ? y : x;
    const int lim = alongx ? d.ny : d.nx;
    for (int k = 1; k <= lp.neg_cells; ++k) {
      const int line = base + sgn * k;
      if ((unsigned)line >= (unsigned)nline) break;  // further rings are outside too
      const int lo = max(0, center - k), hi = min(lim - 1, center + k);
      bool found;
      if (alongx)
        found = ring_line(out.colbits + (int64_t)line * WY, lo, hi, qs, line, d.nx, fmin, fmax,
                          fcount);
      else
        found = ring_line(out.rowbits + (int64_t)line * WX, lo, hi, qs, (int64_t)d.nx * line, 1,
                          fmin, fmax, fcount);
      if (found) break;
    }
  }
  smin[cone][tx] = fcount ? (int32_t)fmin : INT32_MAX;
  smax[cone][tx] = fcount ? (int32_t)fmax : INT32_MIN;
  scnt[cone][tx] = (int32_t)fcount;
  __syncthreads();
  if (cone == 0 && c < cells) {
    int32_t mn = smin[0][tx], mx = smax[0][tx], n = scnt[0][tx];
#pragma unroll
    for (int j = 1; j < 4; ++j) {
      mn = min(mn, smin[j][tx]);
      mx = max(mx, smax[j][tx]);
      n += scnt[j][tx];
    }
    out.neg[c] = (undef && n >= 2 && (int64_t)mx - (int64_t)mn > lp.T_neg) ? 1 : 0;
  }
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
__global__ void __launch_bounds__(256) k_export_layers(const __grid_constant__ CopyJob job) {
  const int l = blockIdx.y;
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
                           const LayerPtrs& out, cudaStream_t st) {
  const int64_t warps = (int64_t)d.nx * d.ny;
  k_columns<<<(unsigned)((warps * 32 + 255) / 256), 256, 0, st>>>(ss, d, lp, out);
  return cudaGetLastError();
}

cudaError_t launch_slope(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                         cudaStream_t st) {
  k_slope<<<cells_blocks(d, 128), 128, 0, st>>>(d, lp, out);
  return cudaGetLastError();
}

cudaError_t launch_negative(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                            cudaStream_t st) {
  k_negative<<<cells_blocks(d, 32), dim3(32, 4), 0, st>>>(d, lp, out);
  return cudaGetLastError();
}

cudaError_t launch_export_layers(const CopyJob& job, cudaStream_t st) {
  int64_t mx = 0;
  for (int l = 0; l < GVOM_LAYER_COUNT; ++l) mx = job.bytes[l] > mx ? job.bytes[l] : mx;
  int64_t blocks = ((mx >> 4) + 255) / 256;
  if (blocks < 1) blocks = 1;
  if (blocks > 148 * 4) blocks = 148 * 4;
  k_export_layers<<<dim3((unsigned)blocks, GVOM_LAYER_COUNT), 256, 0, st>>>(job);
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
