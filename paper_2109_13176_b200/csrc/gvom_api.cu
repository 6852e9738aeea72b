// gvom_api.cu -- host side of the C ABI (include/gvom.h).
//
// Owns no device memory: carves the caller's workspace, validates inputs,
// folds poses into per-sensor affines (reading A4), keeps the buffer ring of
// per-scan maps and enqueues the kernels of k_integrate.cu and
// k_maps.cu on the handle's stream.
#include <math.h>
#include <string.h>

#include <new>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "gvom_internal.cuh"

using namespace gvom;

namespace {
// NVTX range over a host call (SURVEY 5 tracing): names the stage in nsys /
// ncu timelines; a no-op unless a tool is attached (header-only NVTX v3).
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
}  // namespace

namespace {

constexpr size_t kAlign = 256;

inline size_t align_up(size_t x) { return (x + kAlign - 1) & ~(kAlign - 1); }

struct Slot {
  int32_t* lut = nullptr;
  uint32_t* bits = nullptr;
  uint32_t* wprefix = nullptr;
  gvom_voxel* data = nullptr;
  uint32_t* meta = nullptr;  // [0] = k (occupied voxels)
  int64_t origin[3] = {0, 0, 0};
};

struct Layout {
  size_t slot_lut, slot_bits, slot_wprefix, slot_data, slot_meta, slot_stride;
  size_t staging, staging2, outstage, outstage_bytes, rank_tmp, rank_status, epcnt, tilecnt, tilecnt_bytes, layers_f32, layers_u8, qs, defbits, defbits_bytes, mbits, mprefix,
      roll_rows, roll_nmn, roll_bits, total;
  int64_t cap, nblk, cells;
};

int neg_qbits(int nz) {
  int b = 0;
  while ((1 << b) < nz) ++b;
  return 16 + b;
}

bool valid_config(const gvom_config* c) {
  if (!c) return false;
  if (c->nx < 1 || c->ny < 1 || c->nz < 1 || c->nz > 2048) return false;
  if ((int64_t)c->nx * c->ny * c->nz >= (1ll << 31)) return false;
  if (!(c->res > 0) || !isfinite(c->res)) return false;
  if (!(c->z_center_frac >= 0.0 && c->z_center_frac <= 1.0)) return false;
  if (c->buffer_frames < 1 || c->buffer_frames > GVOM_MAX_BUFFER_FRAMES) return false;
  // LUT-direct miss counting: N_m <= points per frame <= 2^30 (A11's cap never binds)
  if (c->max_points_per_frame < 0 || c->max_points_per_frame > (1ll << 30)) return false;
  if (!(c->min_obstacle_height >= 0) || !(c->max_obstacle_height >= c->min_obstacle_height))
    return false;
  if (!(c->density_threshold >= 0.0 && c->density_threshold <= 1.0)) return false;
  if (c->slope_window < 3 || c->slope_window > 9 || (c->slope_window % 2) == 0) return false;
  if (c->min_plane_points < 3) return false;
  if (!(c->neg_obs_threshold >= 0) || c->neg_obs_search_cells < 1) return false;
  // packed cone-sweep keys: (K + 3) << qb < 2^32 with qb = 16 + ceil(log2 nz)
  if ((int64_t)(c->neg_obs_search_cells + 3) << neg_qbits(c->nz) >= (1ll << 32)) return false;
  // the cone sweep's shared-memory ring holds at least two key lines
  if (!neg_sweep_fits(c->nx > c->ny ? c->nx : c->ny, c->neg_obs_search_cells)) return false;
  if (c->flags & ~(GVOM_FLAG_PIPELINE | GVOM_FLAG_SLOPE_SKIP_OBSTACLES | GVOM_FLAG_NEG_8CONE |
                   GVOM_FLAG_ROLLING))
    return false;
  // the rolling map replaces the buffer: one scratch frame slot, no pipelining
  if ((c->flags & GVOM_FLAG_ROLLING) &&
      (c->buffer_frames != 1 || (c->flags & GVOM_FLAG_PIPELINE)))
    return false;
  // the 8-cone search's tile (+ K halo) and prefix counts fit in shared memory
  if ((c->flags & GVOM_FLAG_NEG_8CONE) && neg8_smem_bytes(c->neg_obs_search_cells) > kNegSmemMax)
    return false;
  return true;
}

Dims make_dims(const gvom_config* c) {
  Dims d;
  d.nx = c->nx;
  d.ny = c->ny;
  d.nz = c->nz;
  d.V = (int64_t)c->nx * c->ny * c->nz;
  d.W = (d.V + 31) / 32;
  d.sms = 148;
  d.l2_bytes = 126500000;
  return d;
}

Layout make_layout(const gvom_config* c) {
  Layout l{};
  const Dims d = make_dims(c);
  l.cap = c->max_points_per_frame < d.V ? c->max_points_per_frame : d.V;
  l.nblk = rank_blocks(d);
  l.cells = (int64_t)c->nx * c->ny;
  size_t off = 0;
  l.slot_lut = 0;
  l.slot_bits = align_up(4 * (size_t)d.V);
  l.slot_wprefix = l.slot_bits + align_up(4 * (size_t)d.W);
  l.slot_data = l.slot_wprefix + align_up(4 * (size_t)d.W);
  l.slot_meta = l.slot_data + align_up(sizeof(gvom_voxel) * (size_t)(l.cap > 0 ? l.cap : 1));
  l.slot_stride = l.slot_meta + kAlign;
  // one spare slot when pipelined: integrate(t+1) writes it while
  // compute_maps(t) still reads the K newest
  // one spare slot when pipelined: integrate(t+1) writes it while
  // compute_maps(t) still reads the K newest
  off = l.slot_stride * (size_t)(c->buffer_frames + ((c->flags & GVOM_FLAG_PIPELINE) ? 1 : 0));
  l.staging = off;
  off += align_up(16 * (size_t)(c->max_points_per_frame > 0 ? c->max_points_per_frame : 1));
  // pipelined: a second staging buffer, so the copy of scan t+1 (copy stream)
  // overlaps the integrate of scan t, which still reads the first
  l.staging2 = off;
  if (c->flags & GVOM_FLAG_PIPELINE)
    off += align_up(16 * (size_t)(c->max_points_per_frame > 0 ? c->max_points_per_frame : 1));
  // pipelined gvom_step with pinned host outputs: two device copies of the
  // layers (one export kernel into one, the copy-out stream drains it while
  // the next step's map processing runs)
  l.outstage = off;
  l.outstage_bytes = 0;
  if (c->flags & GVOM_FLAG_PIPELINE) {
    l.outstage_bytes = 5 * align_up(4 * (size_t)c->nx * c->ny) + 3 * align_up((size_t)c->nx * c->ny);
    off += 2 * l.outstage_bytes;
  }
  l.rank_tmp = off;
  off += align_up(4 * (size_t)(l.nblk + 2));
  l.rank_status = off;  // [0] ticket counter, [1 + b] tile status (decoupled look-back)
  off += align_up(8 * (size_t)(l.nblk + 1));
  l.epcnt = off;  // slab partition: per-destination record counts and cursors
  off += align_up(4 * 2 * (size_t)GVOM_MAX_RANKS);
  l.tilecnt = off;  // per finalize tile: occupancy counts, offsets; then the done counter
  l.tilecnt_bytes = align_up(4 * (size_t)(2 * n_tiles(d) + 4));
  off += l.tilecnt_bytes;
  l.layers_f32 = off;  // height, density, slope, rough, cost, spread
  off += 6 * align_up(4 * (size_t)l.cells);
  l.layers_u8 = off;  // hard, soft, neg
  off += 3 * align_up((size_t)l.cells);
  l.qs = off;
  off += align_up(4 * (size_t)l.cells);
  l.defbits = off;  // nmin, nmax, negA, negB, negAT, negBT (cone sweeps)
  l.defbits_bytes = 6 * align_up(4 * (size_t)l.cells);
  off += l.defbits_bytes;
  l.mbits = off;
  off += align_up(4 * (size_t)d.W);
  l.mprefix = off;
  off += align_up(4 * (size_t)d.W);
  if (c->flags & GVOM_FLAG_ROLLING) {  // the window map (k_roll.cu)
    l.roll_rows = off;  // hits, misses, m1, m2: four u64 arrays
    off += 4 * align_up(8 * (size_t)d.V);
    l.roll_nmn = off;
    off += align_up(4 * (size_t)d.V);
    l.roll_bits = off;
    off += align_up(4 * (size_t)d.W);
  }
  l.total = off;
  return l;
}

struct TimedRec {
  int stage;
  cudaEvent_t a, b;
};

}  // namespace

struct gvom_handle {
  gvom_config cfg;
  Dims d;
  Layout lay;
  cudaStream_t st = nullptr;
  char* ws = nullptr;
  std::vector<Slot> slots;
  int K = 0, head = 0, count = 0;
  float4* staging = nullptr;
  uint32_t* rank_tmp = nullptr;
  LayerPtrs layers{};
  uint32_t* mbits = nullptr;
  uint32_t* mprefix = nullptr;
  LayerParams lp{};
  int64_t origin[3] = {0, 0, 0};
  int64_t map_origin[3] = {0, 0, 0};
  bool maps_valid = false;
  // the negative layer's per-cell decision deferred into the export (whole-map
  // sweeps): pending until an export / costmap needs it (ensure_neg)
  bool neg_pending = false;
  SlotSet map_slots{};
  bool timing = false;
  std::vector<TimedRec> recs;
  std::vector<cudaEvent_t> pool;
  int64_t launches = 0;
  uint64_t rank_calls = 0;  // decoupled look-back epochs / ticket base
  uint32_t timing_mask = 0;  // stages bracketed by CUDA events
  TileCounts tc{};
  // slab partition: occupancy built by gvom_slab_occupancy, pending finalize
  PeerMap pm{};  // gvom_set_peers: the other ranks' workspaces (slab partition)
  int32_t slab_y0 = -1, slab_y1 = -1;
  int64_t slab_k = 0;  // occupied voxels of the pending slab
  // fork/join: the cone search runs on `aux` while k_slope runs on `st`
  cudaStream_t aux = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  // pipelined mode (GVOM_FLAG_PIPELINE): map processing on its own stream
  bool pipelined = false;
  int NS = 0;                       // physical slots: K (+1 when pipelined)
  cudaStream_t mst = nullptr;       // map stream (pipelined)
  cudaEvent_t ev_integrated = nullptr;
  // gvom_step with pinned host points: their H2D on the copy stream into
  // staging buffer b (alternating), fenced by ev_staged[b] (copy done) and
  // ev_sfree[b] (the integrate that read buffer b done)
  cudaStream_t cst = nullptr;
  float4* staging2 = nullptr;
  cudaEvent_t ev_staged[2] = {}, ev_sfree[2] = {};
  int stage_parity = 0;
  // ... and pinned host outputs: exported into device buffer b, drained to
  // the host on the copy-out stream (ev_out_ready[b] / ev_out_free[b])
  cudaStream_t cst2 = nullptr;
  char* outstage = nullptr;
  cudaEvent_t ev_out_ready[2] = {}, ev_out_free[2] = {};
  int out_parity = 0;
  static constexpr int kMapsRing = 4;
  cudaEvent_t ev_maps[kMapsRing] = {};
  int64_t maps_calls = 0;           // compute_maps calls so far
  std::vector<int64_t> slot_reader; // last compute_maps call that read a slot
  // gvom_step: the frame's launches, captured and replayed as one CUDA graph
  bool rolling = false;                // GVOM_FLAG_ROLLING: the window map
  RollGrid roll{};
  cudaGraphExec_t gexec = nullptr;
  cudaStream_t cap = nullptr;          // capture stream (the caller's may be legacy)
  // pipelined handles: the map-processing half of a step is a second graph,
  // launched on the map stream; cross-step fences are external event nodes
  cudaGraphExec_t gexec_maps = nullptr;
  cudaStream_t cap_maps = nullptr;
  bool capturing = false;              // inside gvom_step's capture
  int64_t graph_stats[3] = {0, 0, 0};  // graph launches, instantiations, eager steps
  int32_t fault = 0;                   // gvom_debug_inject_fault (tests)
  cudaStream_t ms() const { return pipelined ? mst : st; }
};

namespace {

cudaEvent_t take_event(gvom_handle* h) {
  if (!h->pool.empty()) {
    cudaEvent_t e = h->pool.back();
    h->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  if (cudaEventCreate(&e) != cudaSuccess) return nullptr;
  return e;
}

// Run one stage (a kernel launch or a copy) with optional event timing.
template <class F>
cudaError_t stage(gvom_handle* h, int id, bool is_kernel, F&& f, cudaStream_t on = nullptr) {
  cudaEvent_t a = nullptr, b = nullptr;
  const bool timed = h->timing && ((h->timing_mask >> id) & 1u);
  cudaStream_t ts = on ? on : h->st;
  if (timed) {
    a = take_event(h);
    b = take_event(h);
    // under capture: external event-record nodes, recorded at every replay
    if (a) cudaEventRecordWithFlags(a, ts, h->capturing ? cudaEventRecordExternal : 0u);
  }
  const cudaError_t e = f();
  if (timed && a && b) {
    cudaEventRecordWithFlags(b, ts, h->capturing ? cudaEventRecordExternal : 0u);
    h->recs.push_back({id, a, b});
  }
  if (is_kernel && e == cudaSuccess) h->launches++;
  return e;
}

// Event bracket around a whole call (GVOM_STAGE_INTEGRATE / _MAPS): times the
// call's launches as they run back to back (inside a step graph too), without
// the per-launch events of the kernel stages.
struct Bracket {
  gvom_handle* h;
  int id;
  cudaStream_t s;
  cudaEvent_t a = nullptr;
  Bracket(gvom_handle* h_, int id_, cudaStream_t s_) : h(h_), id(id_), s(s_) {
    if (h->timing && ((h->timing_mask >> id) & 1u)) {
      a = take_event(h);
      if (a) cudaEventRecordWithFlags(a, s, h->capturing ? cudaEventRecordExternal : 0u);
    }
  }
  void end() {
    if (!a) return;
    cudaEvent_t b = take_event(h);
    if (b) {
      cudaEventRecordWithFlags(b, s, h->capturing ? cudaEventRecordExternal : 0u);
      h->recs.push_back({id, a, b});
    } else {
      h->pool.push_back(a);
    }
    a = nullptr;
  }
  ~Bracket() {
    if (a) h->pool.push_back(a);  // the call failed: no record
  }
};

void snap(const gvom_config& c, const double p[3], int64_t o[3]) {
  // reading A3: o = floor(p/res + 0.5) - (nx/2, ny/2, floor(nz * frac))
  o[0] = (int64_t)floor(p[0] / c.res + 0.5) - (int64_t)(c.nx / 2);
  o[1] = (int64_t)floor(p[1] / c.res + 0.5) - (int64_t)(c.ny / 2);
  o[2] = (int64_t)floor(p[2] / c.res + 0.5) - (int64_t)floor((double)c.nz * c.z_center_frac);
}

bool pose_ok(const double* P) {
  for (int i = 0; i < 12; ++i)
    if (!isfinite(P[i])) return false;
  // R R^T = I within 1e-6, det(R) = +1 within 1e-6
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) {
      double s = 0;
      for (int k = 0; k < 3; ++k) s += P[4 * i + k] * P[4 * j + k];
      if (fabs(s - (i == j ? 1.0 : 0.0)) > 1e-6) return false;
    }
  const double det = P[0] * (P[5] * P[10] - P[6] * P[9]) - P[1] * (P[4] * P[10] - P[6] * P[8]) +
                     P[2] * (P[4] * P[9] - P[5] * P[8]);
  return fabs(det - 1.0) <= 1e-6;
}

SensorParams sensor_params(const gvom_config& c, const double* P, const int64_t o[3]) {
  SensorParams sp;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) sp.A[3 * i + j] = (float)(P[4 * i + j] / c.res);
    sp.b[i] = (float)(P[4 * i + 3] / c.res - (double)o[i]);
    sp.S[i] = (int32_t)floorf(sp.b[i]);
  }
  return sp;
}

// the rolling map's window origin and its per-axis physical offsets
void roll_set_origin(RollGrid& g, const gvom_config& c, const int64_t o[3]) {
  auto pm = [](int64_t a, int n) { return (int32_t)(((a % n) + n) % n); };
  g.ox = o[0];
  g.oy = o[1];
  g.oz = o[2];
  g.xo = pm(o[0], c.nx);
  g.yo = pm(o[1], c.ny);
  g.zo = pm(o[2], c.nz);
}

// Memory type of a pointer (cudaPointerGetAttributes).  Within one gvom_step
// call (MemoScope) the answers are memoised -- the call checks the same scan
// and output pointers several times, and the caller keeps every buffer valid
// for the duration of the call -- and the handle's own workspace is device
// memory without asking.
struct PtrMemo {
  static constexpr int kN = 48;
  const void* p[kN];
  int t[kN];
  int n = 0;
  const char* ws0 = nullptr;
  const char* ws1 = nullptr;
  bool on = false;
};
thread_local PtrMemo g_memo;

struct MemoScope {
  explicit MemoScope(const gvom_handle* h) {
    g_memo.on = true;
    g_memo.n = 0;
    g_memo.ws0 = h->ws;
    g_memo.ws1 = h->ws + h->lay.total;
  }
  ~MemoScope() {
    g_memo.on = false;
    g_memo.n = 0;
  }
};

int mem_type(const void* p) {
  if (g_memo.on) {
    const char* c = (const char*)p;
    if (c >= g_memo.ws0 && c < g_memo.ws1) return cudaMemoryTypeDevice;
    for (int i = 0; i < g_memo.n; ++i)
      if (g_memo.p[i] == p) return g_memo.t[i];
  }
  int t = cudaMemoryTypeUnregistered;
  cudaPointerAttributes attr;
  if (cudaPointerGetAttributes(&attr, p) != cudaSuccess)
    cudaGetLastError();
  else
    t = (int)attr.type;
  if (g_memo.on && g_memo.n < PtrMemo::kN) {
    g_memo.p[g_memo.n] = p;
    g_memo.t[g_memo.n] = t;
    g_memo.n++;
  }
  return t;
}

bool is_pinned_host_ptr(const void* p) { return mem_type(p) == cudaMemoryTypeHost; }

bool is_device_ptr(const void* p) {
  const int t = mem_type(p);
  return t == cudaMemoryTypeDevice || t == cudaMemoryTypeManaged;
}

#define GVOM_CU(x)                                     \
  do {                                                 \
    if ((x) != cudaSuccess) return GVOM_E_CUDA;        \
  } while (0)

// rank of the occupied voxels of `bits` -> absolute per-word prefix; k -> *total
cudaError_t run_rank(gvom_handle* h, const uint32_t* bits, uint32_t* wprefix, uint32_t* total) {
  uint64_t* st = (uint64_t*)(h->ws + h->lay.rank_status);
  const uint64_t call = h->rank_calls++;
  const uint32_t epoch = (uint32_t)((call % 0x7ffffffeull) + 1);
  if (epoch == 1 && call > 0) {  // epoch wrapped: clear stale tile status
    cudaError_t e = cudaMemsetAsync(st + 1, 0, 8 * (size_t)h->lay.nblk, h->st);
    if (e != cudaSuccess) return e;
  }
  return launch_rank(bits, h->d, wprefix, st + 1, (unsigned long long*)st,
                     call * (uint64_t)h->lay.nblk, epoch, total, h->st);
}

SlotSet buffer_slots(gvom_handle* h, const int64_t o_out[3]) {
  SlotSet ss{};
  ss.K = h->count;
  ss.kp_log2 = 0;
  while ((1 << ss.kp_log2) < ss.K) ss.kp_log2++;
  for (int age = 0; age < h->count; ++age) {
    const int idx = ((h->head - 1 - age) % h->NS + h->NS) % h->NS;
    const Slot& s = h->slots[idx];
    SlotView& v = ss.s[age];
    h->slot_reader[idx] = h->maps_calls;  // this compute_maps reads the slot
    v.lut = s.lut;
    v.bits = s.bits;
    v.wprefix = s.wprefix;
    v.data = s.data;
    v.dx = (int32_t)(o_out[0] - s.origin[0]);
    v.dy = (int32_t)(o_out[1] - s.origin[1]);
    v.dz = (int32_t)(o_out[2] - s.origin[2]);
    // slots shifted by a whole map extent or more contribute nothing
    if (llabs(o_out[0] - s.origin[0]) >= h->cfg.nx || llabs(o_out[1] - s.origin[1]) >= h->cfg.ny ||
        llabs(o_out[2] - s.origin[2]) >= h->cfg.nz) {
      v.dx = h->cfg.nx;  // every source column out of range
      v.dy = 0;
      v.dz = 0;
    }
  }
  return ss;
}

// Host-side state a step advances while its launches are captured (the ring
// head and count, slot origins, the map-processing bookkeeping).  Restored
// when the capture, instantiation or graph launch fails: none of the captured
// work ran, so the ring must not name a slot whose frame was never written.
struct HostState {
  int head = 0, count = 0;
  std::vector<int64_t> slot_origin;
  std::vector<int64_t> slot_reader;
  int64_t maps_calls = 0, map_origin[3] = {0, 0, 0}, o_z = 0;
  bool maps_valid = false;
  SlotSet map_slots{};
  uint64_t rank_calls = 0;
  bool neg_pending = false;
};

HostState save_state(const gvom_handle* h) {
  HostState s;
  s.head = h->head;
  s.count = h->count;
  for (const Slot& sl : h->slots) s.slot_origin.insert(s.slot_origin.end(), sl.origin, sl.origin + 3);
  s.slot_reader = h->slot_reader;
  s.maps_calls = h->maps_calls;
  for (int i = 0; i < 3; ++i) s.map_origin[i] = h->map_origin[i];
  s.o_z = h->lp.o_z;
  s.maps_valid = h->maps_valid;
  s.map_slots = h->map_slots;
  s.rank_calls = h->rank_calls;
  s.neg_pending = h->neg_pending;
  return s;
}

void restore_state(gvom_handle* h, const HostState& s) {
  h->head = s.head;
  h->count = s.count;
  for (size_t k = 0; k < h->slots.size(); ++k)
    for (int i = 0; i < 3; ++i) h->slots[k].origin[i] = s.slot_origin[3 * k + i];
  h->slot_reader = s.slot_reader;
  h->maps_calls = s.maps_calls;
  for (int i = 0; i < 3; ++i) h->map_origin[i] = s.map_origin[i];
  h->lp.o_z = s.o_z;
  h->maps_valid = s.maps_valid;
  h->map_slots = s.map_slots;
  h->rank_calls = s.rank_calls;
  h->neg_pending = s.neg_pending;
}

// Capture body()'s launches with *role (h->st or h->mst) redirected to a
// private stream (the caller's may be the legacy default stream, which
// cannot be captured), patch them into *gexec (cudaGraphExecUpdate: same
// topology, new kernel arguments) or instantiate anew, and launch the graph
// on the role's real stream.
template <class F>
gvom_status capture_launch(gvom_handle* h, cudaStream_t* role, cudaStream_t* cap,
                                  cudaGraphExec_t* gexec, F&& body) {
  if (!*cap) GVOM_CU(cudaStreamCreateWithFlags(cap, cudaStreamNonBlocking));
  cudaStream_t real = *role;
  const HostState saved = save_state(h);
  GVOM_CU(cudaStreamBeginCapture(*cap, cudaStreamCaptureModeThreadLocal));
  *role = *cap;
  h->capturing = true;
  const gvom_status fs = body();
  h->capturing = false;
  cudaGraph_t g = nullptr;
  cudaError_t ce = cudaStreamEndCapture(*cap, &g);
  *role = real;
  if (h->fault == GVOM_FAULT_CAPTURE) {  // test hook: as if EndCapture had failed
    h->fault = 0;
    ce = cudaErrorStreamCaptureInvalidated;
  }
  if (fs != GVOM_OK || ce != cudaSuccess) {
    if (g) cudaGraphDestroy(g);
    restore_state(h, saved);
    return fs != GVOM_OK ? fs : GVOM_E_CUDA;
  }
  if (*gexec) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(*gexec, g, &info) != cudaSuccess) {
      cudaGetLastError();  // topology changed: instantiate anew
      cudaGraphExecDestroy(*gexec);
      *gexec = nullptr;
    }
  }
  cudaError_t e = cudaSuccess;
  if (!*gexec) {
    e = cudaGraphInstantiate(gexec, g, 0);
    if (e == cudaSuccess) h->graph_stats[1]++;
  }
  cudaGraphDestroy(g);
  if (e == cudaSuccess) e = cudaGraphLaunch(*gexec, real);
  if (e != cudaSuccess) {
    cudaGetLastError();
    restore_state(h, saved);
    return GVOM_E_CUDA;
  }
  return GVOM_OK;
}

}  // namespace

extern "C" {

int32_t gvom_abi_version(void) { return GVOM_ABI_VERSION; }

const char* gvom_status_string(gvom_status s) {
  switch (s) {
    case GVOM_OK: return "ok";
    case GVOM_E_INVALID: return "invalid argument";
    case GVOM_E_NOMEM: return "workspace too small";
    case GVOM_E_CUDA: return "CUDA error";
    case GVOM_E_SENSOR_OUTSIDE: return "sensor outside the map";
    case GVOM_E_EMPTY: return "empty map buffer";
    case GVOM_E_SIZE: return "capacity too small";
  }
  return "unknown status";
}

size_t gvom_workspace_bytes(const gvom_config* cfg) {
  if (!valid_config(cfg)) return 0;
  return make_layout(cfg).total;
}

gvom_status gvom_create(const gvom_config* cfg, void* d_workspace, size_t ws_bytes,
                        void* cuda_stream, gvom_handle** out) {
  if (!out) return GVOM_E_INVALID;
  *out = nullptr;
  if (!valid_config(cfg) || !d_workspace) return GVOM_E_INVALID;
  if (((uintptr_t)d_workspace % kAlign) != 0) return GVOM_E_INVALID;
  const Layout lay = make_layout(cfg);
  if (ws_bytes < lay.total) return GVOM_E_NOMEM;
  gvom_handle* h = new (std::nothrow) gvom_handle();
  if (!h) return GVOM_E_NOMEM;
  h->cfg = *cfg;
  h->d = make_dims(cfg);
  {  // the current device's SM count and L2 size (launch heuristics)
    int dev = 0, v = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) {
      if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && v > 0)
        h->d.sms = v;
      if (cudaDeviceGetAttribute(&v, cudaDevAttrL2CacheSize, dev) == cudaSuccess && v > 0)
        h->d.l2_bytes = v;
    }
    cudaGetLastError();
  }
  h->lay = lay;
  h->st = (cudaStream_t)cuda_stream;
  h->ws = (char*)d_workspace;
  h->K = cfg->buffer_frames;
  h->pipelined = (cfg->flags & GVOM_FLAG_PIPELINE) != 0;
  h->NS = h->K + (h->pipelined ? 1 : 0);
  h->slots.resize(h->NS);
  h->slot_reader.assign(h->NS, -1);
  for (int k = 0; k < h->NS; ++k) {
    char* b = h->ws + lay.slot_stride * (size_t)k;
    Slot& s = h->slots[k];
    s.lut = (int32_t*)(b + lay.slot_lut);
    s.bits = (uint32_t*)(b + lay.slot_bits);
    s.wprefix = (uint32_t*)(b + lay.slot_wprefix);
    s.data = (gvom_voxel*)(b + lay.slot_data);
    s.meta = (uint32_t*)(b + lay.slot_meta);
  }
  h->staging = (float4*)(h->ws + lay.staging);
  h->staging2 = (float4*)(h->ws + lay.staging2);
  h->outstage = h->ws + lay.outstage;
  h->rank_tmp = (uint32_t*)(h->ws + lay.rank_tmp);
  const size_t f32 = align_up(4 * (size_t)lay.cells), u8 = align_up((size_t)lay.cells);
  h->layers.height = (float*)(h->ws + lay.layers_f32);
  h->layers.density = (float*)(h->ws + lay.layers_f32 + f32);
  h->layers.slope = (float*)(h->ws + lay.layers_f32 + 2 * f32);
  h->layers.rough = (float*)(h->ws + lay.layers_f32 + 3 * f32);
  h->layers.cost = (float*)(h->ws + lay.layers_f32 + 4 * f32);
  h->layers.spread = (float*)(h->ws + lay.layers_f32 + 5 * f32);
  h->layers.hard = (uint8_t*)(h->ws + lay.layers_u8);
  h->layers.soft = (uint8_t*)(h->ws + lay.layers_u8 + u8);
  h->layers.neg = (uint8_t*)(h->ws + lay.layers_u8 + 2 * u8);
  h->layers.qs = (int32_t*)(h->ws + lay.qs);
  {
    const size_t c4 = align_up(4 * (size_t)lay.cells);
    char* b = h->ws + lay.defbits;
    h->layers.nmin = (int32_t*)b;
    h->layers.nmax = (int32_t*)(b + c4);
    h->layers.negA = (uint32_t*)(b + 2 * c4);
    h->layers.negB = (uint32_t*)(b + 3 * c4);
    h->layers.negAT = (uint32_t*)(b + 4 * c4);
    h->layers.negBT = (uint32_t*)(b + 5 * c4);
  }
  h->mbits = (uint32_t*)(h->ws + lay.mbits);
  h->tc.tile = (uint32_t*)(h->ws + lay.tilecnt);
  h->tc.offset = h->tc.tile + n_tiles(h->d);
  h->tc.done = h->tc.offset + n_tiles(h->d);
  h->mprefix = (uint32_t*)(h->ws + lay.mprefix);
  // integer thresholds
  h->lp.T_lo = llround(cfg->min_obstacle_height / cfg->res * 65536.0);
  h->lp.T_hi = llround(cfg->max_obstacle_height / cfg->res * 65536.0);
  h->lp.tau = llround(cfg->density_threshold * 65536.0);
  h->lp.T_neg = llround(cfg->neg_obs_threshold / cfg->res * 65536.0);
  h->lp.res = cfg->res;
  h->lp.slope_window = cfg->slope_window;
  h->lp.min_plane_points = cfg->min_plane_points;
  h->lp.neg_cells = cfg->neg_obs_search_cells;
  h->lp.neg_qb = neg_qbits(cfg->nz);
  h->lp.skip_obstacles = (cfg->flags & GVOM_FLAG_SLOPE_SKIP_OBSTACLES) ? 1 : 0;
  h->lp.neg_8cone = (cfg->flags & GVOM_FLAG_NEG_8CONE) ? 1 : 0;
  h->lp.row0 = 0;
  h->lp.row1 = cfg->ny;
  const double zero[3] = {0, 0, 0};
  snap(*cfg, zero, h->origin);
  h->rolling = (cfg->flags & GVOM_FLAG_ROLLING) != 0;
  if (h->rolling) {  // all-zero workspace = the empty window map
    const size_t a8 = align_up(8 * (size_t)h->d.V);
    h->roll.hits = (uint64_t*)(h->ws + lay.roll_rows);
    h->roll.misses = (uint64_t*)(h->ws + lay.roll_rows + a8);
    h->roll.m1 = (uint64_t*)(h->ws + lay.roll_rows + 2 * a8);
    h->roll.m2 = (uint64_t*)(h->ws + lay.roll_rows + 3 * a8);
    h->roll.nmn = (uint32_t*)(h->ws + lay.roll_nmn);
    h->roll.bits = (uint32_t*)(h->ws + lay.roll_bits);
    roll_set_origin(h->roll, h->cfg, h->origin);
  }
  bool ok = true;
  if (h->pipelined) {
    ok = cudaStreamCreateWithFlags(&h->mst, cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&h->ev_integrated, cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; ok && i < gvom_handle::kMapsRing; ++i)
      ok = cudaEventCreateWithFlags(&h->ev_maps[i], cudaEventDisableTiming) == cudaSuccess;
    ok = ok && cudaStreamCreateWithFlags(&h->cst, cudaStreamNonBlocking) == cudaSuccess &&
         cudaStreamCreateWithFlags(&h->cst2, cudaStreamNonBlocking) == cudaSuccess;
    for (int i = 0; ok && i < 2; ++i)
      ok = cudaEventCreateWithFlags(&h->ev_staged[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&h->ev_sfree[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&h->ev_out_ready[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&h->ev_out_free[i], cudaEventDisableTiming) == cudaSuccess;
  }
  if (!ok || cudaStreamCreateWithFlags(&h->aux, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming) != cudaSuccess ||
      cudaMemsetAsync(h->ws, 0, lay.total, h->st) != cudaSuccess) {
    gvom_destroy(h);
    return GVOM_E_CUDA;
  }
  *out = h;
  return GVOM_OK;
}

gvom_status gvom_destroy(gvom_handle* h) {
  if (!h) return GVOM_E_INVALID;
  // the caller frees the workspace next: let the handle's own streams drain
  // first (the copy, planner and map streams may still be using it)
  cudaStreamSynchronize(h->st);  // (null: the legacy default stream)
  for (cudaStream_t s : {h->mst, h->aux, h->cst, h->cst2})
    if (s) cudaStreamSynchronize(s);
  cudaGetLastError();
  for (auto& r : h->recs) {
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  for (auto e : h->pool) cudaEventDestroy(e);
  if (h->ev_fork) cudaEventDestroy(h->ev_fork);
  if (h->ev_join) cudaEventDestroy(h->ev_join);
  if (h->aux) cudaStreamDestroy(h->aux);
  if (h->ev_integrated) cudaEventDestroy(h->ev_integrated);
  for (auto e : h->ev_maps)
    if (e) cudaEventDestroy(e);
  if (h->mst) cudaStreamDestroy(h->mst);
  for (int i = 0; i < 2; ++i) {
    if (h->ev_staged[i]) cudaEventDestroy(h->ev_staged[i]);
    if (h->ev_sfree[i]) cudaEventDestroy(h->ev_sfree[i]);
    if (h->ev_out_ready[i]) cudaEventDestroy(h->ev_out_ready[i]);
    if (h->ev_out_free[i]) cudaEventDestroy(h->ev_out_free[i]);
  }
  if (h->cst) cudaStreamDestroy(h->cst);
  if (h->cst2) cudaStreamDestroy(h->cst2);
  if (h->gexec) cudaGraphExecDestroy(h->gexec);
  if (h->cap) cudaStreamDestroy(h->cap);
  if (h->gexec_maps) cudaGraphExecDestroy(h->gexec_maps);
  if (h->cap_maps) cudaStreamDestroy(h->cap_maps);
  delete h;
  return GVOM_OK;
}

gvom_status gvom_set_stream(gvom_handle* h, void* cuda_stream) {
  if (!h) return GVOM_E_INVALID;
  h->st = (cudaStream_t)cuda_stream;
  return GVOM_OK;
}

gvom_status gvom_synchronize(gvom_handle* h) {
  if (!h) return GVOM_E_INVALID;
  GVOM_CU(cudaStreamSynchronize(h->st));
  if (h->mst) GVOM_CU(cudaStreamSynchronize(h->mst));
  if (h->cst) GVOM_CU(cudaStreamSynchronize(h->cst));
  if (h->cst2) GVOM_CU(cudaStreamSynchronize(h->cst2));
  return GVOM_OK;
}

gvom_status gvom_shift(gvom_handle* h, const double vehicle_xyz[3], int64_t out_delta[3]) {
  NvtxRange nvtx_("gvom_shift");
  if (!h || !vehicle_xyz) return GVOM_E_INVALID;
  for (int i = 0; i < 3; ++i)
    if (!isfinite(vehicle_xyz[i])) return GVOM_E_INVALID;
  int64_t o[3];
  snap(h->cfg, vehicle_xyz, o);
  if (out_delta)
    for (int i = 0; i < 3; ++i) out_delta[i] = o[i] - h->origin[i];
  if (h->rolling) {
    // the window moves: clear the slabs that enter it (reading B9)
    const int n[3] = {h->cfg.nx, h->cfg.ny, h->cfg.nz};
    roll_set_origin(h->roll, h->cfg, o);
    for (int a = 0; a < 3; ++a) {
      const int64_t dlt = o[a] - h->origin[a];
      if (dlt == 0) continue;
      const int cnt = (int)(dlt > 0 ? (dlt < n[a] ? dlt : n[a]) : (-dlt < n[a] ? -dlt : n[a]));
      const int64_t w0 = dlt > 0 ? o[a] + n[a] - cnt : o[a];
      GVOM_CU(stage(h, GVOM_STAGE_MEMSET, true,
                    [&] { return launch_roll_clear(h->roll, h->d, a, w0, cnt, h->st); }));
    }
  }
  for (int i = 0; i < 3; ++i) h->origin[i] = o[i];
  return GVOM_OK;
}

// Validate a frame's scans and fold their poses (A4); sensor voxels in grid (A9).
static gvom_status prepare_scans(gvom_handle* h, const gvom_scan* scans, int32_t n_scans,
                                 SensorParams* sp) {
  if (!h || n_scans < 0 || n_scans > GVOM_MAX_SENSORS || (n_scans > 0 && !scans))
    return GVOM_E_INVALID;
  int64_t total = 0;
  for (int i = 0; i < n_scans; ++i) {
    const gvom_scan& s = scans[i];
    if (s.n < 0 || (s.n > 0 && !s.xyzw) || s.rings < 0) return GVOM_E_INVALID;
    if (((uintptr_t)s.xyzw % 16) != 0) return GVOM_E_INVALID;
    if (!pose_ok(s.sensor_to_world)) return GVOM_E_INVALID;
    sp[i] = sensor_params(h->cfg, s.sensor_to_world, h->origin);
    total += s.n;
  }
  if (total > h->cfg.max_points_per_frame) return GVOM_E_SIZE;
  for (int i = 0; i < n_scans; ++i) {
    const SensorParams& p = sp[i];
    if ((unsigned)p.S[0] >= (unsigned)h->d.nx || (unsigned)p.S[1] >= (unsigned)h->d.ny ||
        (unsigned)p.S[2] >= (unsigned)h->d.nz || !isfinite(p.b[0]) || !isfinite(p.b[1]) ||
        !isfinite(p.b[2]))
      return GVOM_E_SENSOR_OUTSIDE;
  }
  return GVOM_OK;
}

// Device pointers of the scans' points (host points are staged, stream-ordered).
static gvom_status stage_points(gvom_handle* h, const gvom_scan* scans, int32_t n_scans,
                                std::vector<const float4*>& dptr) {
  dptr.assign(n_scans, nullptr);
  int64_t off = 0;
  for (int i = 0; i < n_scans; ++i) {
    const gvom_scan& s = scans[i];
    if (s.n == 0) continue;
    if (is_device_ptr(s.xyzw)) {
      dptr[i] = (const float4*)s.xyzw;
    } else {
      float4* dst = h->staging + off;
      GVOM_CU(stage(h, GVOM_STAGE_H2D, false, [&] {
        return cudaMemcpyAsync(dst, s.xyzw, 16 * (size_t)s.n, cudaMemcpyHostToDevice, h->st);
      }));
      dptr[i] = dst;
      off += s.n;
    }
  }
  return GVOM_OK;
}

// Pipelined mode: before integrate overwrites slot j, the main stream waits
// for the last compute_maps that read it (or a later one: same map stream).
static cudaError_t wait_slot_readers(gvom_handle* h, int j) {
  if (!h->pipelined || h->slot_reader[j] < 0) return cudaSuccess;
  int64_t r = h->slot_reader[j];
  if (h->maps_calls - r > gvom_handle::kMapsRing) r = h->maps_calls - gvom_handle::kMapsRing;
  // under gvom_step's capture: an external wait node (the event is recorded by
  // an earlier step's map-processing graph)
  return cudaStreamWaitEvent(h->st, h->ev_maps[r % gvom_handle::kMapsRing],
                             h->capturing ? cudaEventWaitExternal : 0u);
}

// Ray cast a frame: sensors with the same ring count are batched (up to
// kRayBatch) into one launch with interleaved azimuth tiles.
// Sensors with equal ring counts go into one batch (one ray-cast launch and
// one endpoint launch each, their 32-column tiles interleaved).
static std::vector<RayBatch> ray_batches(const gvom_scan* scans, int32_t n_scans,
                                         const std::vector<const float4*>& dptr,
                                         const SensorParams* sp) {
  std::vector<RayBatch> batches;
  for (int i = 0; i < n_scans; ++i) {
    if (scans[i].n == 0) continue;
    const int32_t rings = scans[i].rings > 1 ? scans[i].rings : 0;
    RayBatch* b = nullptr;
    for (auto& x : batches)
      if (x.rings == rings && x.S < kRayBatch) b = &x;
    if (!b) {
      batches.emplace_back();
      b = &batches.back();
      b->S = 0;
      b->rings = rings;
      b->tile_threads = rings > 1 ? 32 * (int64_t)rings : 32;
    }
    b->pts[b->S] = dptr[i];
    b->n[b->S] = scans[i].n;
    b->sp[b->S] = sp[i];
    b->S++;
  }
  return batches;
}

static cudaError_t raycast_frame(gvom_handle* h, const std::vector<RayBatch>& batches,
                                 uint32_t* miss, uint32_t* bits, const TileCounts& tc,
                                 const SlabRange* slab = nullptr, bool lut_direct = false) {
  for (size_t k = 0; k < batches.size(); ++k) {
    const cudaError_t e = stage(h, GVOM_STAGE_RAYCAST, true, [&] {
      return launch_raycast(batches[k], h->d, miss, bits, tc, k + 1 == batches.size(), h->st,
                            slab, lut_direct);
    });
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// integrate_scan over the rows [slab.y0, slab.y1) (the whole map, or a rank's
// slab in the ray-segment partition)
static gvom_status integrate_rows(gvom_handle* h, const gvom_scan* scans, int32_t n_scans,
                                  const SlabRange& slab) {
  SensorParams sp[GVOM_MAX_SENSORS];
  const gvom_status ps = prepare_scans(h, scans, n_scans, sp);
  if (ps != GVOM_OK) return ps;
  Slot& slot = h->slots[h->head];
  const Dims& d = h->d;
  GVOM_CU(wait_slot_readers(h, h->head));
  Bracket br(h, GVOM_STAGE_INTEGRATE, h->st);
  int64_t t0, t1;  // the tiles of the rows integrated
  slab_tile_range(d, slab, &t0, &t1);
  // pass 0: the slot's LUT to -1 (empty, no misses), its bits cleared.  (Doing
  // this for the next scan right after an integrate, on a side stream beside
  // compute_maps, measured no gain: the reset then competes with k_columns for
  // bandwidth -- c2 step 119.7 vs 119.1 us.)
  GVOM_CU(stage(h, GVOM_STAGE_MEMSET, true,
                [&] { return launch_reset_slot(slot.lut, slot.bits, d, t0, t1, h->st); }));
  // pass 2a: ray tracing, misses counted down in the slot's LUT (LUT-direct)
  TileCounts tc = h->tc;
  tc.total = slot.meta;
  std::vector<const float4*> dptr;
  {
    const gvom_status st = stage_points(h, scans, n_scans, dptr);
    if (st != GVOM_OK) return st;
  }
  const std::vector<RayBatch> batches = ray_batches(scans, n_scans, dptr, sp);
  const bool part = slab.y0 > 0 || slab.y1 < h->cfg.ny;
  GVOM_CU(raycast_frame(h, batches, (uint32_t*)slot.lut, slot.bits, tc, part ? &slab : nullptr,
                        true));
  if (batches.empty())  // no ray-cast launch scanned the (all zero) tile counts
    GVOM_CU(stage(h, GVOM_STAGE_MEMSET, false, [&] {
      return cudaMemsetAsync(tc.offset, 0, 4 * (size_t)n_tiles(d), h->st);
    }));
  // pass 1: ranks of the occupied voxels in L order -> LUT entries + data rows
  GVOM_CU(stage(h, GVOM_STAGE_FINALIZE, true, [&] {
    return launch_finalize_lut(slot.lut, slot.bits, slot.wprefix, slot.data, tc, d, t0, t1,
                               h->st);
  }));
  // pass 2b: per-return metrics into the data rows, one launch per batch
  for (const RayBatch& b : batches)
    GVOM_CU(stage(h, GVOM_STAGE_ENDPOINT, true,
                  [&] { return launch_endpoint(b, d, slot.lut, slot.data, h->st, slab); }));
  // staging buffer 0 read by this call: a later gvom_step's copy into it waits
  if (h->cst && !h->capturing)
    for (int i = 0; i < n_scans; ++i)
      if (dptr[i] && (const void*)dptr[i] != (const void*)scans[i].xyzw) {
        GVOM_CU(cudaEventRecord(h->ev_sfree[0], h->st));
        break;
      }
  for (int i = 0; i < 3; ++i) slot.origin[i] = h->origin[i];
  if (h->rolling)  // the frame map joins the window map (reading B9)
    GVOM_CU(stage(h, GVOM_STAGE_FINALIZE, true, [&] {
      return launch_roll_accumulate(h->roll, d, slot.lut, slot.data, h->st);
    }));
  br.end();
  h->head = (h->head + 1) % h->NS;
  if (h->count < h->K) h->count++;
  if (h->pipelined)
    GVOM_CU(cudaEventRecordWithFlags(h->ev_integrated, h->st,
                                     h->capturing ? cudaEventRecordExternal : 0u));
  return GVOM_OK;
}

gvom_status gvom_integrate_scan(gvom_handle* h, const gvom_scan* scans, int32_t n_scans) {
  NvtxRange nvtx_("gvom_integrate_scan");
  if (!h) return GVOM_E_INVALID;
  return integrate_rows(h, scans, n_scans, SlabRange{0, h->cfg.ny});
}

gvom_status gvom_integrate_slab(gvom_handle* h, const gvom_scan* scans, int32_t n_scans,
                                int32_t y0, int32_t y1) {
  NvtxRange nvtx_("gvom_integrate_slab");
  if (!h || h->pipelined || h->rolling || y0 < 0 || y1 > h->cfg.ny || y0 >= y1)
    return GVOM_E_INVALID;
  return integrate_rows(h, scans, n_scans, SlabRange{y0, y1});
}

// Layers from the surface: the cone search (+ Delta-H decision) on the aux
// stream concurrently with the plane fits on the main stream (fork / join).
static cudaError_t surface_layers(gvom_handle* h) {
  cudaError_t e = cudaEventRecord(h->ev_fork, h->ms());
  if (e == cudaSuccess) e = cudaStreamWaitEvent(h->aux, h->ev_fork, 0);
  if (e == cudaSuccess && h->lp.neg_8cone) {
    h->neg_pending = false;
    e = stage(h, GVOM_STAGE_NEGATIVE, true,
              [&] { return launch_negative8(h->d, h->lp, h->layers, h->aux); }, h->aux);
  } else if (e == cudaSuccess) {
    // whole map: the per-cell decision (k_neg_decide) is made by the export,
    // after the join, which reads the sweeps' min / max on its way (ensure_neg
    // for the other consumers); GVOM_NEG_DEFER=0 decides here (A/B)
    static int defer_env = -1;
    if (defer_env < 0) {
      const char* ev = getenv("GVOM_NEG_DEFER");
      defer_env = ev ? (atoi(ev) ? 1 : 0) : 1;
    }
    const bool defer = defer_env && h->lp.row0 == 0 && h->lp.row1 == h->cfg.ny;
    e = stage(h, GVOM_STAGE_NEGATIVE, true,
              [&] { return launch_negative(h->d, h->lp, h->layers, h->aux, !defer); }, h->aux);
    if (e == cudaSuccess && !defer) h->launches++;  // k_neg_decide
    h->neg_pending = e == cudaSuccess && defer;
  }
  if (e == cudaSuccess)
    e = stage(
        h, GVOM_STAGE_SLOPE, true, [&] { return launch_slope(h->d, h->lp, h->layers, h->ms()); },
        h->ms());
  if (e == cudaSuccess) e = cudaEventRecord(h->ev_join, h->aux);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(h->ms(), h->ev_join, 0);
  return e;
}

gvom_status gvom_compute_maps(gvom_handle* h) {
  NvtxRange nvtx_("gvom_compute_maps");
  if (!h) return GVOM_E_INVALID;
  if (h->count == 0) return GVOM_E_EMPTY;
  const int newest = (h->head - 1 + h->NS) % h->NS;
  int64_t o[3];
  for (int i = 0; i < 3; ++i) o[i] = h->rolling ? h->origin[i] : h->slots[newest].origin[i];
  if (h->pipelined)
    GVOM_CU(cudaStreamWaitEvent(h->mst, h->ev_integrated,
                                h->capturing ? cudaEventWaitExternal : 0u));
  h->lp.o_z = o[2];
  h->lp.row0 = 0;  // every row
  h->lp.row1 = h->cfg.ny;
  Bracket br(h, GVOM_STAGE_MAPS, h->ms());
  if (h->rolling) {  // the window map at the current origin (reading B9)
    GVOM_CU(stage(h, GVOM_STAGE_COLUMNS, true,
                  [&] { return launch_columns_roll(h->roll, h->d, h->lp, h->layers, h->st); }));
  } else {
    h->map_slots = buffer_slots(h, o);
    GVOM_CU(stage(
        h, GVOM_STAGE_COLUMNS, true,
        [&] { return launch_columns(h->map_slots, h->d, h->lp, h->layers, h->ms()); }, h->ms()));
  }
  GVOM_CU(surface_layers(h));
  br.end();
  if (h->pipelined)
    GVOM_CU(cudaEventRecordWithFlags(h->ev_maps[h->maps_calls % gvom_handle::kMapsRing], h->mst,
                                     h->capturing ? cudaEventRecordExternal : 0u));
  h->maps_calls++;
  for (int i = 0; i < 3; ++i) h->map_origin[i] = o[i];
  h->maps_valid = true;
  return GVOM_OK;
}

// A deferred negative decision, before anything other than the one-kernel
// export reads the negative layer (whole map: rows 0..ny).
static cudaError_t ensure_neg(gvom_handle* h) {
  if (!h->neg_pending) return cudaSuccess;
  LayerParams lp = h->lp;
  lp.row0 = 0;
  lp.row1 = h->cfg.ny;
  const cudaError_t e = stage(
      h, GVOM_STAGE_NEGATIVE, true, [&] { return launch_neg_decide(h->d, lp, h->layers, h->ms()); },
      h->ms());
  if (e == cudaSuccess) h->neg_pending = false;
  return e;
}

static const void* layer_src(gvom_handle* h, int layer, size_t* elem) {
  *elem = 4;
  switch (layer) {
    case GVOM_LAYER_HEIGHT: return h->layers.height;
    case GVOM_LAYER_DENSITY: return h->layers.density;
    case GVOM_LAYER_SLOPE: return h->layers.slope;
    case GVOM_LAYER_ROUGHNESS: return h->layers.rough;
    case GVOM_LAYER_HARD: *elem = 1; return h->layers.hard;
    case GVOM_LAYER_SOFT: *elem = 1; return h->layers.soft;
    case GVOM_LAYER_NEGATIVE: *elem = 1; return h->layers.neg;
    case GVOM_LAYER_SPREAD: return h->layers.spread;
    default: return nullptr;
  }
}

gvom_status gvom_export_layers(gvom_handle* h, void* const dst[GVOM_LAYER_COUNT],
                               const size_t dst_bytes[GVOM_LAYER_COUNT]) {
  NvtxRange nvtx_("gvom_export_layers");
  if (!h || !dst || !dst_bytes) return GVOM_E_INVALID;
  if (!h->maps_valid) return GVOM_E_EMPTY;
  CopyJob job;
  bool one_kernel = true;
  for (int l = 0; l < GVOM_LAYER_COUNT; ++l) {
    size_t elem;
    job.src[l] = layer_src(h, l, &elem);
    job.dst[l] = dst[l];
    job.bytes[l] = (int64_t)(elem * (size_t)h->lay.cells);
    if (!dst[l]) return GVOM_E_INVALID;
    if (dst_bytes[l] < (size_t)job.bytes[l]) return GVOM_E_SIZE;
    if (((uintptr_t)dst[l] & 15) != 0 || !is_device_ptr(dst[l])) one_kernel = false;
  }
  if (one_kernel) {  // (with a deferred negative decision made on the way)
    NegDecide dec{};
    if (h->neg_pending && ((uintptr_t)dst[GVOM_LAYER_NEGATIVE] & 3) == 0) {
      dec.qs = h->layers.qs;
      dec.nmin = h->layers.nmin;
      dec.nmax = h->layers.nmax;
      dec.neg = h->layers.neg;
      dec.T_neg = h->lp.T_neg;
      dec.on = true;
    } else {
      GVOM_CU(ensure_neg(h));
    }
    GVOM_CU(stage(
        h, GVOM_STAGE_EXPORT, true, [&] { return launch_export_layers(job, h->ms(), dec); },
        h->ms()));
    h->neg_pending = false;
    return GVOM_OK;
  }
  GVOM_CU(ensure_neg(h));
  for (int l = 0; l < GVOM_LAYER_COUNT; ++l) {
    GVOM_CU(stage(h, GVOM_STAGE_EXPORT, false, [&] {
      return cudaMemcpyAsync(job.dst[l], job.src[l], (size_t)job.bytes[l], cudaMemcpyDefault,
                             h->ms());
    }, h->ms()));
  }
  return GVOM_OK;
}

// One scan end to end (shift + integrate + compute_maps + export): the host
// work is done first (inputs validated before anything is enqueued), then the
// frame's launches are captured on the handle's stream, patched into the cached
// executable graph (cudaGraphExecUpdate: same topology, new kernel arguments)
// or instantiated anew, and launched as one graph.
gvom_status gvom_step(gvom_handle* h, const double vehicle_xyz[3], const gvom_scan* scans,
                      int32_t n_scans, void* const dst[GVOM_LAYER_COUNT],
                      const size_t dst_bytes[GVOM_LAYER_COUNT], const float cost_weights[7],
                      void* cost_dst, size_t cost_bytes, int64_t out_delta[3]) {
  NvtxRange nvtx_("gvom_step");
  if (!h || !vehicle_xyz) return GVOM_E_INVALID;
  MemoScope memo_(h);
  if (dst && !dst_bytes) return GVOM_E_INVALID;
  if ((cost_weights == nullptr) != (cost_dst == nullptr)) return GVOM_E_INVALID;
  if (cost_weights) {
    for (int i = 0; i < 7; ++i)
      if (!isfinite(cost_weights[i])) return GVOM_E_INVALID;
    if (cost_bytes < 4 * (size_t)h->lay.cells) return GVOM_E_SIZE;
  }
  if (dst)
    for (int l = 0; l < GVOM_LAYER_COUNT; ++l) {
      size_t elem;
      layer_src(h, l, &elem);
      if (!dst[l]) return GVOM_E_INVALID;
      if (dst_bytes[l] < elem * (size_t)h->lay.cells) return GVOM_E_SIZE;
    }
  const gvom_status ss = gvom_shift(h, vehicle_xyz, out_delta);
  if (ss != GVOM_OK) return ss;
  {
    SensorParams sp[GVOM_MAX_SENSORS];
    const gvom_status ps = prepare_scans(h, scans, n_scans, sp);
    if (ps != GVOM_OK) return ps;
  }
  // capture needs stream-ordered work only: points and outputs on the device
  // or in pinned host memory (stage-timing events and the pipelined fences
  // become external event nodes), and a stream that is not already being
  // captured by the caller
  bool graph = true;
  for (int i = 0; graph && i < n_scans; ++i)
    if (scans[i].n > 0 && !is_device_ptr(scans[i].xyzw) && !is_pinned_host_ptr(scans[i].xyzw))
      graph = false;
  for (int l = 0; graph && dst && l < GVOM_LAYER_COUNT; ++l)  // pageable outputs too
    if (!is_device_ptr(dst[l]) && !is_pinned_host_ptr(dst[l])) graph = false;
  if (graph && cost_dst && !is_device_ptr(cost_dst) && !is_pinned_host_ptr(cost_dst))
    graph = false;
  if (graph) {
    cudaStreamCaptureStatus cs;
    GVOM_CU(cudaStreamIsCapturing(h->st, &cs));
    graph = cs == cudaStreamCaptureStatusNone;
  }
  auto integrate = [&]() -> gvom_status { return gvom_integrate_scan(h, scans, n_scans); };
  auto maps = [&]() -> gvom_status {
    gvom_status s = gvom_compute_maps(h);
    if (s == GVOM_OK && dst && cost_weights)
      s = gvom_export_layers_cost(h, dst, dst_bytes, cost_weights, cost_dst, cost_bytes);
    else if (s == GVOM_OK && dst)
      s = gvom_export_layers(h, dst, dst_bytes);
    else if (s == GVOM_OK && cost_weights)
      s = gvom_costmap(h, cost_weights, cost_dst, cost_bytes);
    return s;
  };
  if (!graph) {
    h->graph_stats[2]++;
    const gvom_status s = integrate();
    return s == GVOM_OK ? maps() : s;
  }
  if (!h->pipelined) {  // one graph on the handle's stream
    const gvom_status s = capture_launch(h, &h->st, &h->cap, &h->gexec, [&] {
      const gvom_status si = integrate();
      return si == GVOM_OK ? maps() : si;
    });
    if (s == GVOM_OK) h->graph_stats[0]++;
    return s;
  }
  // pipelined: integrate on the handle's stream, map processing + export on
  // the map stream, each its own graph (the fences between steps are the
  // external event nodes recorded / waited inside them).  Pinned host points
  // are copied on the copy stream into the staging buffer the integrate
  // before last read (ev_sfree), so the copy overlaps the previous scan's
  // integrate; the integrate graph waits for it (ev_staged).
  gvom_scan dsc[GVOM_MAX_SENSORS];
  int b = -1;
  for (int i = 0; i < n_scans; ++i)
    if (scans[i].n > 0 && !is_device_ptr(scans[i].xyzw)) b = h->stage_parity;
  if (b >= 0) {
    float4* buf = b ? h->staging2 : h->staging;
    GVOM_CU(cudaStreamWaitEvent(h->cst, h->ev_sfree[b], 0));
    int64_t off = 0;
    for (int i = 0; i < n_scans; ++i) {
      dsc[i] = scans[i];
      if (scans[i].n > 0 && !is_device_ptr(scans[i].xyzw)) {
        GVOM_CU(stage(h, GVOM_STAGE_H2D, false, [&] {
          return cudaMemcpyAsync(buf + off, scans[i].xyzw, 16 * (size_t)scans[i].n,
                                 cudaMemcpyHostToDevice, h->cst);
        }, h->cst));
        dsc[i].xyzw = (const float*)(buf + off);
        off += scans[i].n;
      }
    }
    GVOM_CU(cudaEventRecord(h->ev_staged[b], h->cst));
    h->stage_parity ^= 1;
  }
  auto integrate_staged = [&]() -> gvom_status {
    if (b < 0) return integrate();
    GVOM_CU(cudaStreamWaitEvent(h->st, h->ev_staged[b], cudaEventWaitExternal));
    const gvom_status si = gvom_integrate_scan(h, dsc, n_scans);
    if (si == GVOM_OK)
      GVOM_CU(cudaEventRecordWithFlags(h->ev_sfree[b], h->st, cudaEventRecordExternal));
    return si;
  };
  gvom_status s = capture_launch(h, &h->st, &h->cap, &h->gexec, integrate_staged);
  // pinned host outputs (no costmap): the map graph exports into device buffer
  // ob (after the copy-out of the step before last drained it) and the
  // copy-out stream moves it to the host, so the next step's map processing
  // does not wait for the device-to-host copies
  bool host_out = dst && !cost_weights;
  for (int l = 0; host_out && l < GVOM_LAYER_COUNT; ++l)
    if (!is_pinned_host_ptr(dst[l])) host_out = false;
  if (host_out) {
    const int ob = h->out_parity;
    void* sdst[GVOM_LAYER_COUNT];
    size_t sbytes[GVOM_LAYER_COUNT];
    char* p = h->outstage + (size_t)ob * h->lay.outstage_bytes;
    for (int l = 0; l < GVOM_LAYER_COUNT; ++l) {
      size_t elem;
      layer_src(h, l, &elem);
      sdst[l] = p;
      sbytes[l] = elem * (size_t)h->lay.cells;
      p += align_up(sbytes[l]);
    }
    auto maps_staged = [&]() -> gvom_status {
      gvom_status sm = gvom_compute_maps(h);
      if (sm != GVOM_OK) return sm;
      GVOM_CU(cudaStreamWaitEvent(h->mst, h->ev_out_free[ob], cudaEventWaitExternal));
      sm = gvom_export_layers(h, sdst, sbytes);
      if (sm == GVOM_OK)
        GVOM_CU(cudaEventRecordWithFlags(h->ev_out_ready[ob], h->mst, cudaEventRecordExternal));
      return sm;
    };
    if (s == GVOM_OK) s = capture_launch(h, &h->mst, &h->cap_maps, &h->gexec_maps, maps_staged);
    if (s == GVOM_OK) {
      GVOM_CU(cudaStreamWaitEvent(h->cst2, h->ev_out_ready[ob], 0));
      for (int l = 0; l < GVOM_LAYER_COUNT; ++l)
        GVOM_CU(stage(h, GVOM_STAGE_EXPORT, false, [&] {
          return cudaMemcpyAsync(dst[l], sdst[l], sbytes[l], cudaMemcpyDeviceToHost, h->cst2);
        }, h->cst2));
      GVOM_CU(cudaEventRecord(h->ev_out_free[ob], h->cst2));
      h->out_parity ^= 1;
      h->graph_stats[0]++;
    }
    return s;
  }
  if (s == GVOM_OK) s = capture_launch(h, &h->mst, &h->cap_maps, &h->gexec_maps, maps);
  if (s == GVOM_OK) h->graph_stats[0]++;
  return s;
}

gvom_status gvom_debug_inject_fault(gvom_handle* h, int32_t what) {
  if (!h || (what != 0 && what != GVOM_FAULT_CAPTURE)) return GVOM_E_INVALID;
  h->fault = what;
  return GVOM_OK;
}

gvom_status gvom_graph_stats(gvom_handle* h, int64_t out[3]) {
  if (!h || !out) return GVOM_E_INVALID;
  for (int i = 0; i < 3; ++i) out[i] = h->graph_stats[i];
  return GVOM_OK;
}

gvom_status gvom_export_2d(gvom_handle* h, gvom_layer layer, void* dst, size_t dst_bytes) {
  NvtxRange nvtx_("gvom_export_2d");
  if (!h || !dst) return GVOM_E_INVALID;
  if (!h->maps_valid) return GVOM_E_EMPTY;
  size_t elem;
  const void* src = layer_src(h, (int)layer, &elem);
  if (!src) return GVOM_E_INVALID;
  const size_t bytes = elem * (size_t)h->lay.cells;
  if (dst_bytes < bytes) return GVOM_E_SIZE;
  if (layer == GVOM_LAYER_NEGATIVE) GVOM_CU(ensure_neg(h));
  GVOM_CU(stage(h, GVOM_STAGE_EXPORT, false, [&] {
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, h->ms());
  }));
  return GVOM_OK;
}

gvom_status gvom_costmap(gvom_handle* h, const float weights[7], void* dst, size_t dst_bytes) {
  NvtxRange nvtx_("gvom_costmap");
  if (!h || !weights || !dst) return GVOM_E_INVALID;
  if (!h->maps_valid) return GVOM_E_EMPTY;
  const size_t bytes = 4 * (size_t)h->lay.cells;
  if (dst_bytes < bytes) return GVOM_E_SIZE;
  CostWeights cw;
  for (int i = 0; i < 7; ++i) {
    if (!isfinite(weights[i])) return GVOM_E_INVALID;
    cw.w[i] = weights[i];
  }
  const bool direct = is_device_ptr(dst) && ((uintptr_t)dst & 3) == 0;
  float* out = direct ? (float*)dst : h->layers.cost;
  GVOM_CU(ensure_neg(h));
  GVOM_CU(stage(
      h, GVOM_STAGE_EXPORT, true,
      [&] { return launch_costmap(h->d, h->layers, cw, out, h->ms()); }, h->ms()));
  if (!direct)
    GVOM_CU(cudaMemcpyAsync(dst, out, bytes, cudaMemcpyDefault, h->ms()));
  return GVOM_OK;
}

gvom_status gvom_export_layers_cost(gvom_handle* h, void* const dst[GVOM_LAYER_COUNT],
                                   const size_t dst_bytes[GVOM_LAYER_COUNT],
                                   const float weights[7], void* cost_dst, size_t cost_bytes) {
  NvtxRange nvtx_("gvom_export_layers_cost");
  if (!h || !dst || !dst_bytes || !weights || !cost_dst) return GVOM_E_INVALID;
  if (!h->maps_valid) return GVOM_E_EMPTY;
  CostWeights cw;
  for (int i = 0; i < 7; ++i) {
    if (!isfinite(weights[i])) return GVOM_E_INVALID;
    cw.w[i] = weights[i];
  }
  if (cost_bytes < 4 * (size_t)h->lay.cells) return GVOM_E_SIZE;
  GVOM_CU(ensure_neg(h));
  CopyJob job;
  bool fused = is_device_ptr(cost_dst) && ((uintptr_t)cost_dst & 3) == 0;
  for (int l = 0; l < GVOM_LAYER_COUNT; ++l) {
    size_t elem;
    job.src[l] = layer_src(h, l, &elem);
    job.dst[l] = dst[l];
    job.bytes[l] = (int64_t)(elem * (size_t)h->lay.cells);
    if (!dst[l]) return GVOM_E_INVALID;
    if (dst_bytes[l] < (size_t)job.bytes[l]) return GVOM_E_SIZE;
    if (((uintptr_t)dst[l] & 3) != 0 || !is_device_ptr(dst[l])) fused = false;
  }
  if (!fused) {  // host (or unaligned) destinations: copies + the costmap kernel
    const gvom_status s = gvom_export_layers(h, dst, dst_bytes);
    return s != GVOM_OK ? s : gvom_costmap(h, weights, cost_dst, cost_bytes);
  }
  GVOM_CU(stage(
      h, GVOM_STAGE_EXPORT, true,
      [&] { return launch_export_cost(h->d, h->layers, job, cw, (float*)cost_dst, h->ms()); },
      h->ms()));
  return GVOM_OK;
}

gvom_status gvom_export_window(gvom_handle* h, uint64_t* d_hits, uint64_t* d_misses,
                               uint32_t* d_min_dz, uint64_t* d_m1, uint64_t* d_m2) {
  if (!h || !d_hits || !d_misses || !d_min_dz || !d_m1 || !d_m2) return GVOM_E_INVALID;
  if (!h->rolling) return GVOM_E_INVALID;
  GVOM_CU(stage(h, GVOM_STAGE_EXPORT, true, [&] {
    return launch_roll_export(h->roll, h->d, d_hits, d_misses, d_min_dz, d_m1, d_m2, h->st);
  }));
  return GVOM_OK;
}

gvom_status gvom_map_origin(gvom_handle* h, int64_t out_origin[3]) {
  if (!h || !out_origin) return GVOM_E_INVALID;
  if (!h->maps_valid) return GVOM_E_EMPTY;
  for (int i = 0; i < 3; ++i) out_origin[i] = h->map_origin[i];
  return GVOM_OK;
}

gvom_status gvom_export_voxels(gvom_handle* h, int32_t* d_lut, gvom_voxel* d_data, int64_t cap,
                               int64_t* out_k) {
  NvtxRange nvtx_("gvom_export_voxels");
  if (!h || !d_lut || !out_k || cap < 0 || (cap > 0 && !d_data)) return GVOM_E_INVALID;
  if (h->rolling) return GVOM_E_INVALID;  // see gvom_export_window
  if (!h->maps_valid) return GVOM_E_EMPTY;
  const Dims& d = h->d;
  if (h->mst) GVOM_CU(cudaStreamSynchronize(h->mst));
  GVOM_CU(cudaMemsetAsync(h->mbits, 0, 4 * (size_t)d.W, h->st));
  GVOM_CU(stage(h, GVOM_STAGE_MERGE, true,
                [&] { return launch_merge_bits(h->map_slots, d, h->mbits, h->st); }));
  uint32_t* ktot = h->rank_tmp + h->lay.nblk;
  GVOM_CU(stage(h, GVOM_STAGE_MERGE, true,
                [&] { return run_rank(h, h->mbits, h->mprefix, ktot); }));
  uint32_t k = 0;
  GVOM_CU(cudaMemcpyAsync(&k, ktot, 4, cudaMemcpyDeviceToHost, h->st));
  GVOM_CU(cudaStreamSynchronize(h->st));
  *out_k = k;
  if ((int64_t)k > cap) return GVOM_E_SIZE;
  GVOM_CU(stage(h, GVOM_STAGE_MERGE, true, [&] {
    return launch_merge_write(h->map_slots, d, h->mbits, h->mprefix, d_lut, d_data, h->st);
  }));
  GVOM_CU(cudaStreamSynchronize(h->st));
  return GVOM_OK;
}

gvom_status gvom_export_frame(gvom_handle* h, int32_t age, int32_t* d_lut, gvom_voxel* d_data,
                              int64_t cap, int64_t* out_k, int64_t out_origin[3]) {
  if (!h || !d_lut || !out_k || cap < 0 || (cap > 0 && !d_data)) return GVOM_E_INVALID;
  if (age < 0 || age >= h->count) return GVOM_E_EMPTY;
  const int idx = ((h->head - 1 - age) % h->NS + h->NS) % h->NS;
  const Slot& s = h->slots[idx];
  if (h->mst) GVOM_CU(cudaStreamSynchronize(h->mst));
  uint32_t k = 0;
  GVOM_CU(cudaMemcpyAsync(&k, s.meta, 4, cudaMemcpyDeviceToHost, h->st));
  GVOM_CU(cudaStreamSynchronize(h->st));
  *out_k = k;
  if (out_origin)
    for (int i = 0; i < 3; ++i) out_origin[i] = s.origin[i];
  if ((int64_t)k > cap) return GVOM_E_SIZE;
  GVOM_CU(cudaMemcpyAsync(d_lut, s.lut, 4 * (size_t)h->d.V, cudaMemcpyDefault, h->st));
  if (k > 0)
    GVOM_CU(cudaMemcpyAsync(d_data, s.data, sizeof(gvom_voxel) * (size_t)k, cudaMemcpyDefault,
                            h->st));
  GVOM_CU(cudaStreamSynchronize(h->st));
  return GVOM_OK;
}

// ---- multi-GPU slab partition --------------------------------
static bool slab_ok(const gvom_handle* h, int32_t y0, int32_t y1) {
  return h && !h->pipelined && !h->rolling && y0 >= 0 && y1 <= h->cfg.ny && y0 < y1;
}

gvom_status gvom_partial_scan(gvom_handle* h, const gvom_scan* scans, int32_t n_scans,
                              uint32_t* d_miss, gvom_endpoint* d_ep, int64_t ep_cap,
                              const int32_t* slab_y, int32_t n_ranks, int64_t* out_counts) {
  NvtxRange nvtx_("gvom_partial_scan");
  if (!h || !d_miss || !slab_y || !out_counts || n_ranks < 1 || n_ranks > GVOM_MAX_RANKS ||
      ep_cap < 0 || (ep_cap > 0 && !d_ep) || h->rolling)
    return GVOM_E_INVALID;
  SlabBounds sb;
  sb.P = n_ranks;
  for (int r = 0; r <= n_ranks; ++r) sb.y[r] = slab_y[r];
  if (sb.y[0] != 0 || sb.y[n_ranks] != h->cfg.ny) return GVOM_E_INVALID;
  for (int r = 0; r < n_ranks; ++r)
    if (sb.y[r + 1] < sb.y[r]) return GVOM_E_INVALID;
  SensorParams sp[GVOM_MAX_SENSORS];
  const gvom_status ps = prepare_scans(h, scans, n_scans, sp);
  if (ps != GVOM_OK) return ps;
  std::vector<const float4*> dptr;
  {
    const gvom_status st = stage_points(h, scans, n_scans, dptr);
    if (st != GVOM_OK) return st;
  }
  const Dims& d = h->d;
  uint32_t* cnt = (uint32_t*)(h->ws + h->lay.epcnt);
  uint32_t* cur = cnt + GVOM_MAX_RANKS;
  GVOM_CU(cudaMemsetAsync(d_miss, 0, 4 * (size_t)d.V, h->st));
  GVOM_CU(cudaMemsetAsync(cnt, 0, 4 * (size_t)GVOM_MAX_RANKS, h->st));
  TileCounts none{};
  GVOM_CU(raycast_frame(h, ray_batches(scans, n_scans, dptr, sp), d_miss, nullptr, none));
  for (int i = 0; i < n_scans; ++i) {
    const gvom_scan& s = scans[i];
    if (s.n == 0) continue;
    GVOM_CU(stage(h, GVOM_STAGE_ENDPOINT, true,
                  [&] { return launch_ep_count(dptr[i], s.n, sp[i], d, sb, cnt, h->st); }));
  }
  uint32_t hc[GVOM_MAX_RANKS];
  GVOM_CU(cudaMemcpyAsync(hc, cnt, 4 * (size_t)n_ranks, cudaMemcpyDeviceToHost, h->st));
  GVOM_CU(cudaStreamSynchronize(h->st));
  uint32_t ho[GVOM_MAX_RANKS];
  int64_t tot = 0;
  for (int r = 0; r < n_ranks; ++r) {
    ho[r] = (uint32_t)tot;
    tot += hc[r];
    out_counts[r] = hc[r];
  }
  if (tot > ep_cap) return GVOM_E_SIZE;
  GVOM_CU(cudaMemcpyAsync(cur, ho, 4 * (size_t)n_ranks, cudaMemcpyHostToDevice, h->st));
  for (int i = 0; i < n_scans; ++i) {
    const gvom_scan& s = scans[i];
    if (s.n == 0) continue;
    GVOM_CU(stage(h, GVOM_STAGE_ENDPOINT, true, [&] {
      return launch_ep_write(dptr[i], s.n, sp[i], d, sb, cur, (EpRecord*)d_ep, h->st);
    }));
  }
  GVOM_CU(cudaStreamSynchronize(h->st));  // the host buffer ho must outlive the copy
  return GVOM_OK;
}

static void slab_tiles(const gvom_handle* h, int32_t y0, int32_t y1, int64_t* t0, int64_t* t1) {
  const int64_t row = (int64_t)h->cfg.nx * h->cfg.nz;
  *t0 = (y0 * row) >> kTileShift;
  *t1 = ((y1 * row) + (1 << kTileShift) - 1) >> kTileShift;
}

gvom_status gvom_slab_occupancy(gvom_handle* h, int32_t y0, int32_t y1, const gvom_endpoint* d_ep,
                                int64_t n_ep, int64_t* out_k) {
  NvtxRange nvtx_("gvom_slab_occupancy");
  if (!slab_ok(h, y0, y1) || !out_k || n_ep < 0 || (n_ep > 0 && !d_ep)) return GVOM_E_INVALID;
  Slot& slot = h->slots[h->head];
  GVOM_CU(stage(h, GVOM_STAGE_MEMSET, true, [&] {
    return launch_zero3(slot.lut, (size_t)h->lay.slot_bits, slot.bits,
                        (size_t)(h->lay.slot_wprefix - h->lay.slot_bits), h->tc.tile,
                        h->lay.tilecnt_bytes, h->d, h->st);
  }));
  GVOM_CU(stage(h, GVOM_STAGE_RANK_COUNT, true, [&] {
    return launch_slab_bits((const EpRecord*)d_ep, n_ep, slot.bits, h->tc.tile, h->st);
  }));
  int64_t t0, t1;
  slab_tiles(h, y0, y1, &t0, &t1);
  TileCounts tc = h->tc;
  tc.total = slot.meta;
  GVOM_CU(stage(h, GVOM_STAGE_RANK_SCAN, true, [&] { return launch_tile_scan(tc, t0, t1, h->st); }));
  uint32_t k = 0;
  GVOM_CU(cudaMemcpyAsync(&k, slot.meta, 4, cudaMemcpyDeviceToHost, h->st));
  GVOM_CU(cudaStreamSynchronize(h->st));
  *out_k = k;
  h->slab_k = k;
  h->slab_y0 = y0;
  h->slab_y1 = y1;
  return GVOM_OK;
}

// Slab finalize: the slab's miss counts come either from the reduce-scattered
// slab rows (d_miss_slab, copied into the slot) or, fused, from the P ranks'
// partial grids read over peer memory by the finalize itself (peers).
static gvom_status slab_finalize(gvom_handle* h, int32_t y0, int32_t y1,
                                 const uint32_t* d_miss_slab, const PeerGrids* peers,
                                 const gvom_endpoint* d_ep, int64_t n_ep, int64_t base) {
  if (!slab_ok(h, y0, y1) || n_ep < 0 || (n_ep > 0 && !d_ep) || base < 0) return GVOM_E_INVALID;
  if (h->slab_y0 != y0 || h->slab_y1 != y1) return GVOM_E_INVALID;  // occupancy first
  if (base + h->slab_k > h->lay.cap) return GVOM_E_SIZE;  // rows [base, base + k)
  Slot& slot = h->slots[h->head];
  const Dims& d = h->d;
  const int64_t row = (int64_t)h->cfg.nx * h->cfg.nz;
  if (!peers)
    GVOM_CU(stage(h, GVOM_STAGE_MEMSET, false, [&] {
      return cudaMemcpyAsync(slot.lut + y0 * row, d_miss_slab, 4 * (size_t)((y1 - y0) * row),
                             cudaMemcpyDeviceToDevice, h->st);
    }));
  int64_t t0, t1;
  slab_tiles(h, y0, y1, &t0, &t1);
  TileCounts tc = h->tc;
  tc.total = slot.meta;
  GVOM_CU(stage(h, GVOM_STAGE_FINALIZE, true, [&] {
    return launch_finalize_tiles(slot.lut, slot.bits, slot.wprefix, slot.data, tc, d, h->st, t0,
                                 t1, (uint32_t)base, peers);
  }));
  GVOM_CU(stage(h, GVOM_STAGE_ENDPOINT, true, [&] {
    return launch_endpoint_records((const EpRecord*)d_ep, n_ep, slot.lut, slot.data, h->st);
  }));
  // the integrate path expects zero tile counters at rest
  GVOM_CU(stage(h, GVOM_STAGE_MEMSET, false, [&] {
    return cudaMemsetAsync(h->tc.tile, 0, h->lay.tilecnt_bytes, h->st);
  }));
  for (int i = 0; i < 3; ++i) slot.origin[i] = h->origin[i];
  h->head = (h->head + 1) % h->NS;
  if (h->count < h->K) h->count++;
  h->slab_y0 = h->slab_y1 = -1;
  return GVOM_OK;
}

gvom_status gvom_slab_finalize(gvom_handle* h, int32_t y0, int32_t y1, const uint32_t* d_miss_slab,
                               const gvom_endpoint* d_ep, int64_t n_ep, int64_t base) {
  NvtxRange nvtx_("gvom_slab_finalize");
  if (!d_miss_slab) return GVOM_E_INVALID;
  return slab_finalize(h, y0, y1, d_miss_slab, nullptr, d_ep, n_ep, base);
}

gvom_status gvom_slab_finalize_peers(gvom_handle* h, int32_t y0, int32_t y1,
                                     const uint32_t* const* d_miss_grids, int32_t n_grids,
                                     const gvom_endpoint* d_ep, int64_t n_ep, int64_t base) {
  NvtxRange nvtx_("gvom_slab_finalize_peers");
  if (!d_miss_grids || n_grids < 1 || n_grids > GVOM_MAX_RANKS) return GVOM_E_INVALID;
  PeerGrids pg{};
  pg.P = n_grids;
  for (int p = 0; p < n_grids; ++p) {
    if (!d_miss_grids[p] || ((uintptr_t)d_miss_grids[p] & 15) != 0) return GVOM_E_INVALID;
    pg.g[p] = d_miss_grids[p];
  }
  return slab_finalize(h, y0, y1, nullptr, &pg, d_ep, n_ep, base);
}

gvom_status gvom_slot_buffers(gvom_handle* h, int32_t age, int32_t** out_d_lut,
                              gvom_voxel** out_d_data, int64_t* out_cap) {
  if (!h || !out_d_lut || !out_d_data || !out_cap || age < 0 || age >= h->K) return GVOM_E_INVALID;
  const int idx = ((h->head - 1 - age) % h->NS + h->NS) % h->NS;
  *out_d_lut = h->slots[idx].lut;
  *out_d_data = h->slots[idx].data;
  *out_cap = h->lay.cap;
  return GVOM_OK;
}

gvom_status gvom_set_peers(gvom_handle* h, const void* const* d_peer_workspaces,
                           const int32_t* slab_y, int32_t n_ranks, int32_t rank) {
  if (!h || n_ranks < 0 || n_ranks > GVOM_MAX_RANKS) return GVOM_E_INVALID;
  PeerMap pm{};
  if (n_ranks > 0) {
    if (!d_peer_workspaces || !slab_y || rank < 0 || rank >= n_ranks) return GVOM_E_INVALID;
    if (slab_y[0] != 0 || slab_y[n_ranks] != h->cfg.ny) return GVOM_E_INVALID;
    if (d_peer_workspaces[rank] != (const void*)h->ws) return GVOM_E_INVALID;
    pm.P = n_ranks;
    for (int r = 0; r <= n_ranks; ++r) {
      if (r > 0 && slab_y[r] < slab_y[r - 1]) return GVOM_E_INVALID;
      pm.y[r] = slab_y[r];
    }
    for (int r = 0; r < n_ranks; ++r) {
      if (!d_peer_workspaces[r]) return GVOM_E_INVALID;
      pm.delta[r] = (int64_t)((const char*)d_peer_workspaces[r] - h->ws);
    }
  }
  h->pm = pm;
  return GVOM_OK;
}

gvom_status gvom_row_work(gvom_handle* h, int32_t y0, int32_t y1, uint64_t* d_out) {
  NvtxRange nvtx_("gvom_row_work");
  if (!h || h->rolling || !d_out || y0 < 0 || y1 > h->cfg.ny || y0 >= y1) return GVOM_E_INVALID;
  if (h->count == 0) return GVOM_E_EMPTY;
  const Slot& slot = h->slots[(h->head - 1 + h->NS) % h->NS];
  GVOM_CU(stage(h, GVOM_STAGE_EXPORT, true, [&] {
    return launch_row_work(slot.lut, slot.data, h->d, y0, y1, (unsigned long long*)d_out, h->st);
  }));
  return GVOM_OK;
}

gvom_status gvom_slab_complete(gvom_handle* h, int64_t k_total) {
  NvtxRange nvtx_("gvom_slab_complete");
  if (!h || h->pipelined || h->rolling || h->count == 0 || k_total < 0 || k_total > h->lay.cap)
    return GVOM_E_INVALID;
  Slot& slot = h->slots[(h->head - 1 + h->NS) % h->NS];
  GVOM_CU(stage(h, GVOM_STAGE_RANK_COUNT, true, [&] {
    return launch_bits_from_lut(slot.lut, slot.bits, slot.wprefix, h->d, slot.meta,
                                (uint32_t)k_total, h->st);
  }));
  return GVOM_OK;
}

gvom_status gvom_compute_maps_slab(gvom_handle* h, int32_t y0, int32_t y1, int32_t phase) {
  NvtxRange nvtx_("gvom_compute_maps_slab");
  if (!slab_ok(h, y0, y1) || (phase != 0 && phase != 1)) return GVOM_E_INVALID;
  if (h->count == 0) return GVOM_E_EMPTY;
  if (phase == 0) {
    const int newest = (h->head - 1 + h->NS) % h->NS;
    int64_t o[3];
    for (int i = 0; i < 3; ++i) o[i] = h->slots[newest].origin[i];
    h->map_slots = buffer_slots(h, o);
    h->map_slots.pm = h->pm;  // shifted rows of other slabs: their owners' memory
    h->lp.o_z = o[2];
    GVOM_CU(stage(h, GVOM_STAGE_COLUMNS, true, [&] {
      return launch_columns(h->map_slots, h->d, h->lp, h->layers, h->st, (int64_t)y0 * h->cfg.nx,
                            (int64_t)y1 * h->cfg.nx);
    }));
    for (int i = 0; i < 3; ++i) h->map_origin[i] = o[i];
    return GVOM_OK;
  }
  GVOM_CU(stage(h, GVOM_STAGE_NEGATIVE, true,
                [&] { return launch_transpose_init(h->d, h->lp, h->layers, h->st); }));
  // slope / roughness / negative obstacles of the slab's rows only (their
  // windows and cones read the gathered surface rows around them)
  h->lp.row0 = y0;
  h->lp.row1 = y1;
  GVOM_CU(surface_layers(h));
  h->maps_valid = true;
  return GVOM_OK;
}

gvom_status gvom_map_stream(gvom_handle* h, void** out_stream) {
  if (!h || !out_stream) return GVOM_E_INVALID;
  *out_stream = (void*)h->ms();
  return GVOM_OK;
}

gvom_status gvom_surface_buffer(gvom_handle* h, int32_t** out_d_qs) {
  if (!h || !out_d_qs) return GVOM_E_INVALID;
  *out_d_qs = h->layers.qs;
  return GVOM_OK;
}

gvom_status gvom_obstacle_buffers(gvom_handle* h, uint8_t** out_d_hard, uint8_t** out_d_soft) {
  if (!h || !out_d_hard || !out_d_soft) return GVOM_E_INVALID;
  *out_d_hard = h->layers.hard;
  *out_d_soft = h->layers.soft;
  return GVOM_OK;
}

gvom_status gvom_set_timing(gvom_handle* h, int32_t enable) {
  if (!h) return GVOM_E_INVALID;
  h->timing = enable != 0;
  h->timing_mask = enable == -1 ? 0xffffffffu : (uint32_t)enable;
  return GVOM_OK;
}

gvom_status gvom_stage_times(gvom_handle* h, double* out, int32_t n_doubles) {
  if (!h || !out || n_doubles < 2 * GVOM_STAGE_COUNT) return GVOM_E_INVALID;
  for (int i = 0; i < 2 * GVOM_STAGE_COUNT; ++i) out[i] = 0.0;
  GVOM_CU(cudaStreamSynchronize(h->st));
  for (auto& r : h->recs) {
    float ms = 0.f;
    if (cudaEventElapsedTime(&ms, r.a, r.b) == cudaSuccess) {
      out[2 * r.stage] += ms;
      out[2 * r.stage + 1] += 1.0;
    }
    h->pool.push_back(r.a);
    h->pool.push_back(r.b);
  }
  h->recs.clear();
  return GVOM_OK;
}

int64_t gvom_launch_count(const gvom_handle* h) { return h ? h->launches : -1; }

}  // extern "C"
