// gvom_internal.cuh -- shared declarations of the CUDA path (kernels + host).
// Independent of oracle/ (no shared code, headers or tables).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "gvom.h"

namespace gvom {

constexpr int kTileWords = 256;           // finalize tile: 256 words = 8192 voxels
constexpr int kTileShift = 13;            // voxel L -> tile
constexpr int kRankWordsPerBlock = 1024;  // bitmask words per rank tile (32768 voxels)
constexpr int kRankThreads = 256;         // 4 words per thread
constexpr uint32_t kMissSat = 1u << 30;   // A11
constexpr int32_t kQsUndef = INT32_MIN;   // undefined surface sentinel in qs[]

// Per-sensor transform in voxel units (reading A4), folded on the host.
struct SensorParams {
  float A[9];
  float b[3];
  int32_t S[3];  // floor(b), the sensor voxel
};

struct Dims {
  int32_t nx, ny, nz;
  int64_t V;  // nx*ny*nz
  int64_t W;  // bitmask words = ceil(V/32)
  // the device the handle runs on (queried in gvom_create; the B200 values
  // until then): launch heuristics derive their thresholds from these
  int32_t sms;       // multiprocessors (B200: 148)
  int64_t l2_bytes;  // L2 cache size (B200: 126.5 MB)
};

// One buffer map ("lookup array, data array, map origin").
struct SlotView {
  const int32_t* lut;
  const uint32_t* bits;
  const uint32_t* wprefix;
  const gvom_voxel* data;
  int32_t dx, dy, dz;  // o_out - o_slot  (source u = v + d)
  int32_t pad;
};

// The ray-segment slab partition with motion (gvom_set_peers): rank r owns
// rows [y[r], y[r+1]) of every buffer map; a shifted older map's rows of other
// slabs are read from their owner's workspace (peer memory) at the same
// offsets, delta[r] bytes from this handle's.  P = 0: everything local.
struct PeerMap {
  int32_t P;
  int32_t y[GVOM_MAX_RANKS + 1];
  int64_t delta[GVOM_MAX_RANKS];
};

struct SlotSet {
  SlotView s[GVOM_MAX_BUFFER_FRAMES];
  int32_t K;
  int32_t kp_log2;  // log2 of the lanes per slot group (pow2 >= K)
  PeerMap pm;
};

// byte offset from this handle's workspace to the owner of row y's (peers)
__host__ __device__ inline int64_t peer_delta(const PeerMap& pm, int y) {
  if (pm.P <= 0) return 0;
  int lo = 0, hi = pm.P - 1;  // slab r with y[r] <= y < y[r+1]
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (pm.y[mid] <= y)
      lo = mid;
    else
      hi = mid - 1;
  }
  return pm.delta[lo];
}
template <class T>
__host__ __device__ inline T* rebase(T* p, int64_t delta) {
  return reinterpret_cast<T*>(reinterpret_cast<char*>(const_cast<void*>(
                                  reinterpret_cast<const void*>(p))) + delta);
}

struct LayerPtrs {
  float* height;
  float* density;
  uint8_t* hard;
  uint8_t* soft;
  uint8_t* neg;
  float* slope;
  float* rough;
  float* cost;    // costmap scratch (gvom_costmap, NEXT-4)
  float* spread;  // variance of the surface voxel's returns (NEXT-3)
  int32_t* qs;    // [ny][nx] fixed-point surface q_s, kQsUndef if undefined
  // cone-sweep keys of the surface (see neg_keys): [ny][nx] and transposed
  // [nx][ny] copies, so that every sweep reads its lines contiguously
  uint32_t* negA;
  uint32_t* negB;
  uint32_t* negAT;
  uint32_t* negBT;
  int32_t* nmin;  // [ny][nx] min / max of the heights found by the cone search
  int32_t* nmax;
};

struct LayerParams {
  int64_t T_lo, T_hi, tau, T_neg;
  double res;
  int64_t o_z;
  int32_t slope_window, min_plane_points, neg_cells;
  int32_t skip_obstacles;  // GVOM_FLAG_SLOPE_SKIP_OBSTACLES
  int32_t neg_8cone;       // GVOM_FLAG_NEG_8CONE
  int32_t neg_qb;          // q_s < 2^neg_qb (= 16 + ceil(log2 nz)); see neg_keys
  // rows [row0, row1) whose slope / roughness / negative-obstacle cells are
  // computed (the whole map, or a rank's slab in phase 1 of the slab path)
  int32_t row0, row1;
};

// Cone-sweep keys (k_negative): a found ring (distance D, heights q) is packed
// as (D << qb) | q for the minimum and (D << qb) | (2^qb - 1 - q) for the
// maximum, so ONE unsigned min over sub-cones yields the least D and, among
// the sub-cones attaining it, the least (resp. greatest) height -- exactly the
// recurrence's tie rule.  An undefined cell is "not found" = (K + 1) << qb.
// gvom_create guarantees (K + 3) << qb < 2^32 (no overflow when adding 1 << qb
// to the not-found key).
__host__ __device__ inline void neg_keys(int32_t q, const LayerParams& lp, uint32_t& ka,
                                         uint32_t& kb) {
  const uint32_t one = 1u << lp.neg_qb;
  if (q == kQsUndef) {
    ka = kb = (uint32_t)(lp.neg_cells + 1) << lp.neg_qb;
  } else {
    ka = one + (uint32_t)q;
    kb = one + (one - 1u - (uint32_t)q);
  }
}

// k_negative shared memory: a ring of R slots, each one key line of A keys and
// one of B keys; the key of cross position bb sits at [neg_guard_left + bb],
// with not-found guards over bb in [-K-1, -1] and [B, B+K] and the TMA
// destination (bb = 0) 16-byte aligned; plus 4 state lines of B + 2K + 2.
constexpr int kNegRing = 32;                                  // max ring slots
constexpr size_t kNegSmemMax = 227 * 1024 - 2 * kNegRing * 8;  // minus mbarriers
__host__ __device__ inline int neg_guard_left(int K) { return (K + 1 + 3) & ~3; }
__host__ __device__ inline int neg_line_stride(int B, int K) {
  return (neg_guard_left(K) + B + K + 1 + 3) & ~3;
}
inline size_t neg_slot_bytes(int B, int K) { return 8 * (size_t)neg_line_stride(B, K); }
inline size_t neg_state_bytes(int B, int K) { return 16 * ((size_t)B + 2 * (size_t)K + 2); }
inline bool neg_sweep_fits(int B, int K) {
  return neg_state_bytes(B, K) + 2 * neg_slot_bytes(B, K) <= kNegSmemMax;
}
// k_negative8 (GVOM_FLAG_NEG_8CONE): a tile (16 or 32 cells square) + K halo
// of q_s (int32), its summed-area table of defined cells (u16) and t_k (u8)
inline size_t neg8_smem_bytes(int K, int tile = 32) {
  const size_t W = (size_t)tile + 2 * (size_t)K, W1 = W + 1;
  return ((4 * W * W + 2 * W1 * W1 + (size_t)K + 1) + 15) & ~(size_t)15;
}

// ---- launchers (each launches exactly one kernel; returns cudaError_t) ----
// Occupancy counts per finalize tile, kept by the ray cast as bits are set;
// the frame's last ray-cast block turns them into exclusive offsets.
struct TileCounts {
  uint32_t* tile;    // [n_tiles] newly occupied voxels per tile
  uint32_t* offset;  // [n_tiles] exclusive prefix of tile
  uint32_t* done;    // [1] finished ray-cast blocks (last-block scan)
  uint32_t* total;   // k of the frame (slot meta), written by the scan
};
__host__ __device__ inline int64_t n_tiles(const Dims& d) {
  return (d.V + (1 << kTileShift) - 1) >> kTileShift;
}

// Up to kRayBatch sensors with the same ring count traced by one launch; their
// 32-column tiles are interleaved (tile t of every sensor, then t+1, ...) so a
// wave of warps covers one azimuth band of all sensors (voxels close together).
constexpr int kRayBatch = 16;
struct RayBatch {
  int32_t S;      // sensors in the batch
  int32_t rings;  // common ring count (<= 1: unstructured, one warp per tile)
  int64_t tile_threads;
  const float4* pts[kRayBatch];
  int64_t n[kRayBatch];
  SensorParams sp[kRayBatch];
};
// Rows [y0, y1) of the map a rank owns (the ray-segment slab partition): the
// ray cast traces only the part of every ray inside them, and only returns
// inside them are binned.  {0, ny} = the whole map.
struct SlabRange {
  int32_t y0, y1;
};
cudaError_t launch_raycast(const RayBatch& rb, const Dims& d, uint32_t* miss_grid,
                           uint32_t* bits, const TileCounts& tc, bool last_launch,
                           cudaStream_t st, const SlabRange* slab = nullptr,
                           bool lut_direct = false);
// rank (from the tile counts) + in-place LUT encode + data-row init, one launch
// the P ranks' partial miss grids, device pointers the GPU can load from
// (peer memory, NEXT-2): the finalize sums them instead of reading lut_inplace
struct PeerGrids {
  const uint32_t* g[GVOM_MAX_RANKS];
  int32_t P;
};
// base: added to every rank (a slab's global rank offset, 0 otherwise)
cudaError_t launch_finalize_tiles(int32_t* lut_inplace, const uint32_t* bits, uint32_t* wprefix,
                                  gvom_voxel* data, const TileCounts& tc, const Dims& d,
                                  cudaStream_t st, int64_t t_begin = 0, int64_t t_end = -1,
                                  uint32_t base = 0, const PeerGrids* peers = nullptr);
// the integrate path (LUT-direct): pass 0 resets the slot's LUT tiles [t0, t1)
// to -1 and clears their bits; the ray cast counts misses down in place; pass 1
// ranks the occupied voxels and initialises their rows (k_finalize_lut)
cudaError_t launch_reset_slot(int32_t* lut, uint32_t* bits, const Dims& d, int64_t t0,
                              int64_t t1, cudaStream_t st);
cudaError_t launch_finalize_lut(int32_t* lut, const uint32_t* bits, uint32_t* wprefix,
                                gvom_voxel* data, const TileCounts& tc, const Dims& d, int64_t t0,
                                int64_t t1, cudaStream_t st);
// tiles [*t0, *t1) holding the voxels of rows [y0, y1)
inline void slab_tile_range(const Dims& d, const SlabRange& s, int64_t* t0, int64_t* t1) {
  const int64_t row = (int64_t)d.nx * d.nz;
  *t0 = ((int64_t)s.y0 * row) >> kTileShift;
  *t1 = (((int64_t)s.y1 * row) + (1 << kTileShift) - 1) >> kTileShift;
}
cudaError_t launch_rank(const uint32_t* bits, const Dims& d, uint32_t* wprefix, uint64_t* status,
                        unsigned long long* ticket, uint64_t base, uint32_t epoch,
                        uint32_t* total, cudaStream_t st);
// zeroes a[0:abytes), b[0:bbytes), c[0:cbytes) (multiples of 16, 16-byte aligned)
cudaError_t launch_zero3(void* a, size_t abytes, void* b, size_t bbytes, void* c, size_t cbytes,
                         const Dims& d, cudaStream_t st);
// per-return hits / min_dz / moments of a sensor batch (same tiling as the ray cast)
cudaError_t launch_endpoint(const RayBatch& rb, const Dims& d, const int32_t* lut,
                            gvom_voxel* data, cudaStream_t st, const SlabRange& slab);
cudaError_t launch_negative8(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                             cudaStream_t st);  // 8-cone variant -> neg directly
cudaError_t launch_columns(const SlotSet& ss, const Dims& d, const LayerParams& lp,
                           const LayerPtrs& out, cudaStream_t st, int64_t cbeg = 0,
                           int64_t cend = -1);
// ---- rolling map (k_roll.cu; GVOM_FLAG_ROLLING, NEXT-3, reading B9) ----
struct RollGrid {
  // per physical voxel P (struct of arrays: a pass-through touches 8 bytes)
  uint64_t* hits;
  uint64_t* misses;
  uint64_t* m1;
  uint64_t* m2;
  uint32_t* nmn;   // ~min_dz (0 = no return)
  uint32_t* bits;  // occupancy (hits >= 1)
  int64_t ox, oy, oz;  // window origin (world voxels); P = (w mod n) per axis
  int32_t xo, yo, zo;  // o mod n: logical x -> physical x + xo (wrapped)
};
cudaError_t launch_roll_clear(const RollGrid& g, const Dims& d, int axis, int64_t w0, int cnt,
                              cudaStream_t st);
cudaError_t launch_roll_accumulate(const RollGrid& g, const Dims& d, const int32_t* lut,
                                   const gvom_voxel* data, cudaStream_t st);
cudaError_t launch_columns_roll(const RollGrid& g, const Dims& d, const LayerParams& lp,
                                const LayerPtrs& out, cudaStream_t st);
cudaError_t launch_roll_export(const RollGrid& g, const Dims& d, uint64_t* hits, uint64_t* misses,
                               uint32_t* min_dz, uint64_t* m1, uint64_t* m2, cudaStream_t st);

// ---- multi-GPU slab partition (k_slab.cu) ----
// out[y] for y in [y0, y1): pass-throughs + returns of row y (slab balancing)
cudaError_t launch_row_work(const int32_t* lut, const gvom_voxel* data, const Dims& d, int32_t y0,
                            int32_t y1, unsigned long long* out, cudaStream_t st);
struct SlabBounds {
  int32_t P;
  int32_t y[GVOM_MAX_RANKS + 1];  // slab r = rows [y[r], y[r+1])
};
struct EpRecord {  // == gvom_endpoint
  uint32_t L, dz;
};
cudaError_t launch_ep_count(const float4* pts, int64_t n, const SensorParams& sp, const Dims& d,
                            const SlabBounds& sb, uint32_t* counts, cudaStream_t st);
cudaError_t launch_ep_write(const float4* pts, int64_t n, const SensorParams& sp, const Dims& d,
                            const SlabBounds& sb, uint32_t* cursor, EpRecord* out,
                            cudaStream_t st);
cudaError_t launch_slab_bits(const EpRecord* ep, int64_t n, uint32_t* bits, uint32_t* tile_counts,
                             cudaStream_t st);
cudaError_t launch_tile_scan(const TileCounts& tc, int64_t t_begin, int64_t t_end,
                             cudaStream_t st);
cudaError_t launch_endpoint_records(const EpRecord* ep, int64_t n, const int32_t* lut,
                                    gvom_voxel* data, cudaStream_t st);
// occupancy bits and per-word rank prefix of a whole slot rebuilt from its
// LUT (after the slabs' LUT rows were all-gathered); *meta = k_total
cudaError_t launch_bits_from_lut(const int32_t* lut, uint32_t* bits, uint32_t* wprefix,
                                 const Dims& d, uint32_t* meta, uint32_t k_total, cudaStream_t st);
cudaError_t launch_transpose_init(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                                  cudaStream_t st);
cudaError_t launch_slope(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                         cudaStream_t st);
cudaError_t launch_negative(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                            cudaStream_t st, bool decide = true);  // cone sweeps -> nmin / nmax (slope writes neg)
cudaError_t launch_merge_bits(const SlotSet& ss, const Dims& d, uint32_t* mbits, cudaStream_t st);
cudaError_t launch_merge_write(const SlotSet& ss, const Dims& d, const uint32_t* mbits,
                               const uint32_t* mprefix, int32_t* lut, gvom_voxel* data,
                               cudaStream_t st);

struct CopyJob {
  const void* src[GVOM_LAYER_COUNT];
  void* dst[GVOM_LAYER_COUNT];
  int64_t bytes[GVOM_LAYER_COUNT];
};
// dec.on: the negative layer (job index GVOM_LAYER_NEGATIVE) is decided from
// the cone sweeps' min / max while it is exported (k_neg_decide fused into
// the export: written to job.dst and to dec.neg)
struct NegDecide {
  const int32_t* qs = nullptr;
  const int32_t* nmin = nullptr;
  const int32_t* nmax = nullptr;
  uint8_t* neg = nullptr;
  int64_t T_neg = 0;
  bool on = false;
};
cudaError_t launch_export_layers(const CopyJob& job, cudaStream_t st,
                                 const NegDecide& dec = NegDecide{});
// k_neg_decide alone over rows [lp.row0, lp.row1) (a deferred decision)
cudaError_t launch_neg_decide(const Dims& d, const LayerParams& lp, const LayerPtrs& out,
                              cudaStream_t st);
struct CostWeights {
  float w[7];  // hard, soft, density, negative, slope, roughness, unknown
};
// all layers to job.dst (device, 4-byte aligned) + the costmap, one pass
cudaError_t launch_export_cost(const Dims& d, const LayerPtrs& in, const CopyJob& job,
                               const CostWeights& cw, float* cost, cudaStream_t st);
cudaError_t launch_costmap(const Dims& d, const LayerPtrs& in, const CostWeights& cw, float* out,
                           cudaStream_t st);

inline int64_t rank_blocks(const Dims& d) {
  return (d.W + kRankWordsPerBlock - 1) / kRankWordsPerBlock;
}

}  // namespace gvom
