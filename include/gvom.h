/*
 * gvom.h -- C ABI of the B200-native G-VOM per-scan voxel-map update.
 *
 * G-VOM: "a GPU accelerated voxel mapping system for off-road navigation"
 * (arXiv 2109.13176, /root/reference/PAPER.md, cited below as P:<line>).
 * The calls follow the paper's problem statement: "Our system requires only
 * odometry and lidar sensor data ... [maps] can then be exported as a series
 * of 2D maps", with a fixed-size map centred on the vehicle.
 *
 * Conventions:
 *  - Every call returns gvom_status (0 = OK); nothing throws or aborts.
 *  - Every device operation is enqueued on the handle's CUDA stream, in call
 *    order; calls return before the GPU finishes unless stated otherwise.
 *  - Pointers are plain host or device addresses (CUDA unified addressing
 *    decides which).  The caller owns every buffer it passes, including the
 *    workspace; the library allocates no device memory of its own.
 *  - Buffers passed to a call must stay valid until the stream has passed
 *    that call (the caller synchronises, e.g. with gvom_synchronize()).
 *  - A handle is not thread-safe; several handles may coexist.
 *  - Voxel units: voxel (x,y,z) of a map with origin o covers world
 *    [(o+v)*res, (o+v+1)*res).  Linear index L = z + nz*(x + nx*y)
 *    (z fastest, then x, then y).  2D layers are [ny][nx], x fastest.
 */
#ifndef GVOM_H
#define GVOM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define GVOM_API __attribute__((visibility("default")))
#else
#define GVOM_API
#endif

#define GVOM_ABI_VERSION 1
#define GVOM_MAX_BUFFER_FRAMES 32
#define GVOM_MAX_SENSORS 64
#define GVOM_MAX_RANKS 64

typedef enum gvom_status {
  GVOM_OK = 0,
  GVOM_E_INVALID = -1,        /* bad argument, config or pose                         */
  GVOM_E_NOMEM = -2,          /* workspace smaller than gvom_workspace_bytes()        */
  GVOM_E_CUDA = -3,           /* a CUDA runtime call failed                           */
  GVOM_E_SENSOR_OUTSIDE = -4, /* a sensor voxel is outside the grid: scan rejected,
                                 map state unchanged (reading A9)                     */
  GVOM_E_EMPTY = -5,          /* compute_maps / export on an empty buffer             */
  GVOM_E_SIZE = -6            /* destination or point capacity too small              */
} gvom_status;

/* Map and layer parameters.  The paper names these but gives values only for
 * the map size and resolution ("typically [256,256,64] with a
 * resolution of 40 cm"); defaults are in DESIGN.md "Parameters". */
/* Pipelined mode ("Both of these processes can be run asynchronously"):
 * map processing (compute_maps, export_2d / export_layers) runs on the
 * handle's own map stream (gvom_map_stream) so integrate_scan of the next scan
 * overlaps compute_maps of this one.  One spare buffer slot is allocated; the
 * slot an integrate overwrites is fenced on the compute_maps that last read
 * it.  Results of compute_maps / exports are ordered on the map stream
 * (except gvom_step's copies to pinned host outputs, see gvom_step).       */
#define GVOM_FLAG_PIPELINE 1
/* SPEC S:338 / SURVEY 8(f) NEXT-3 variant: hard and soft obstacle cells are
 * left out of every slope / roughness window (and get NaN themselves).    */
#define GVOM_FLAG_SLOPE_SKIP_OBSTACLES 2
/* SPEC S:327 / SURVEY 8(f) NEXT-3 variant: the negative-obstacle search uses
 * 8 cones at j*45 degrees with half-angle 22.5 degrees (Chebyshev rings)
 * instead of the paper's 4 axis cones (fig. 4); same decision rule.  The
 * search tile needs about 6 (32 + 2K)^2 bytes of shared memory, so K <= 82
 * (else GVOM_E_INVALID).                                                   */
#define GVOM_FLAG_NEG_8CONE 4
/* SURVEY 8(f) NEXT-3 variant, the rolling map (K = infinity; reading B9):
 * instead of a buffer of K scan maps merged at every compute_maps, ONE window
 * map accumulates every scan (u64 counts) since each voxel entered the
 * window; gvom_shift moves the window, dropping the voxels that leave it and
 * clearing the ones that enter it (stored toroidally in world voxel
 * coordinates: only the entering slabs are written).  compute_maps uses the
 * current window origin.  Requires buffer_frames == 1 (the scratch slot of
 * the scan being integrated) and no GVOM_FLAG_PIPELINE; the slab calls and
 * gvom_export_voxels are unavailable (GVOM_E_INVALID) -- see
 * gvom_export_window.  Extra workspace: 36 bytes per voxel.                */
#define GVOM_FLAG_ROLLING 8

typedef struct gvom_config {
  int32_t nx, ny, nz;            /* voxels, each >= 1, nz <= 2048, nx*ny*nz < 2^31 */
  double res;                    /* metres per voxel edge, > 0                    */
  double z_center_frac;          /* vehicle z at floor(nz*frac) voxels (reading A3)      */
  int32_t buffer_frames;         /* K per-scan maps kept ("the buffer"), 1..32       */
  int32_t flags;                 /* GVOM_FLAG_* (0: default)                              */
  int64_t max_points_per_frame;  /* capacity: points of all sensors of one frame          */
  double min_obstacle_height;    /* metres above the surface                     */
  double max_obstacle_height;    /* metres above the surface                     */
  double density_threshold;      /* hard iff density >= threshold (reading A20)   */
  int32_t slope_window;          /* N of the N x N plane fit, odd, 3..9          */
  int32_t min_plane_points;      /* >= 3 defined cells for a fit (reading A22)           */
  double neg_obs_threshold;      /* Delta-H in metres, flag iff larger    */
  int32_t neg_obs_search_cells;  /* cone search distance K in cells, >= 1, with
                                    (K + 3) * nz' * 65536 < 2^32 (nz' = nz rounded up to a
                                    power of two: packed sweep keys) and
                                    48 * max(nx, ny) + 64 * K < ~227 KiB (the sweep's
                                    shared-memory ring); else GVOM_E_INVALID             */
  int32_t pad1;
} gvom_config;

/* One lidar scan of one sensor ("pointcloud and odometry data").
 * xyzw: n points, float32 [n][4] (x, y, z, ignored) in the SENSOR frame,
 *       16-byte aligned, host (pinned or pageable) or device memory.
 *       Non-finite points and exact (0,0,0) no-returns are dropped (A5).
 * sensor_to_world: 3x4 row-major [R | t] odometry pose, metres; R must be
 *       orthonormal with det +1 within 1e-6 (else GVOM_E_INVALID).
 * rings: points per azimuth column when the scan is in sensor order
 *       (column-major, beam-fastest), or 0 for an unordered cloud.  Only the
 *       work assignment uses it; results do not depend on it.            */
typedef struct gvom_scan {
  const float* xyzw;
  int64_t n;
  double sensor_to_world[12];
  int32_t rings;
  int32_t pad;
} gvom_scan;

/* One data-array row ("number of returns within the voxel, number of
 * rays passing though the voxel, and the height of the lowest return").
 * min_dz: lowest return inside the voxel in 1/65536 voxel above its floor
 * (reading A12); m1 = sum dz, m2 = sum dz^2 over the returns (A13).      */
typedef struct gvom_voxel {
  uint32_t hits;
  uint32_t misses;
  uint32_t min_dz;
  uint32_t reserved;
  uint64_t m1;
  uint64_t m2;
} gvom_voxel;

/* The 2D maps (fig:outputs P:39).  f32 layers use NaN as nodata;
 * flag layers are uint8 0/1.  All [ny][nx], x fastest.                  */
typedef enum gvom_layer {
  GVOM_LAYER_HEIGHT = 0,    /* f32 metres, world z of the surface      */
  GVOM_LAYER_DENSITY = 1,   /* f32 in [0,1], band-weighted density      */
  GVOM_LAYER_HARD = 2,      /* u8 hard positive obstacle                */
  GVOM_LAYER_SOFT = 3,      /* u8 soft positive obstacle                */
  GVOM_LAYER_NEGATIVE = 4,  /* u8 negative obstacle              */
  GVOM_LAYER_SLOPE = 5,     /* f32 radians, atan |grad| of the plane    */
  GVOM_LAYER_ROUGHNESS = 6, /* f32 m^2, mean squared plane residual     */
  GVOM_LAYER_SPREAD = 7,    /* f32 m^2, variance of the returns in the surface
                               voxel from the moments m1, m2 (NEXT-3, A13)     */
  GVOM_LAYER_COUNT = 8
} gvom_layer;

typedef struct gvom_handle gvom_handle;

/* Bytes of device workspace a handle with this config needs (0 if invalid). */
GVOM_API size_t gvom_workspace_bytes(const gvom_config* cfg);

/* Create a handle over a caller-owned device workspace (>= workspace_bytes,
 * 256-byte aligned) on CUDA stream `cuda_stream` (cudaStream_t, may be NULL
 * for the legacy default stream).  Initialises the workspace on the stream.
 * The initial origin is the snap of vehicle (0,0,0).                       */
GVOM_API gvom_status gvom_create(const gvom_config* cfg, void* d_workspace, size_t ws_bytes,
                        void* cuda_stream, gvom_handle** out);
/* gvom_destroy waits for the handle's work (its stream and internal streams)
 * before releasing its driver objects, so the workspace may be freed after. */
GVOM_API gvom_status gvom_destroy(gvom_handle* h);
GVOM_API gvom_status gvom_set_stream(gvom_handle* h, void* cuda_stream);
GVOM_API gvom_status gvom_synchronize(gvom_handle* h);

/* Re-centre the map on the vehicle ("fixed map size centered on the
 * vehicle"; P:81 origin "always an integer multiple of the map resolution").
 * o = floor(p/res + 0.5) - (nx/2, ny/2, floor(nz*z_center_frac)) voxels
 * (reading A3).  Sets the origin used by subsequent integrate_scan calls;
 * writes o_new - o_old to out_delta_voxels (may be NULL).  Host only, except
 * with GVOM_FLAG_ROLLING, where it also enqueues the clearing of the
 * entering slabs of the window map on the handle's stream.                */
GVOM_API gvom_status gvom_shift(gvom_handle* h, const double vehicle_xyz[3], int64_t out_delta_voxels[3]);

/* Pointcloud processing: transform the scans of n_scans sensors into
 * the map frame, bin the returns (LUT + data array), trace every ray from its
 * sensor to its return counting pass-throughs, and insert the resulting map
 * (LUT, data array, origin) into the buffer, evicting the oldest when K maps
 * are held.  All sensors of one call form one buffer map (reading A15).
 * Errors: GVOM_E_INVALID (pose, n < 0, n_scans outside 0..64),
 * GVOM_E_SIZE (sum n > max_points_per_frame), GVOM_E_SENSOR_OUTSIDE (scan
 * rejected, state unchanged).  n_scans = 0 pushes an empty map.    */
GVOM_API gvom_status gvom_integrate_scan(gvom_handle* h, const gvom_scan* scans, int32_t n_scans);

/* The ray-segment slab partition (multi-GPU, DESIGN.md
 * section 8): gvom_integrate_scan restricted to the map rows [y0, y1) that
 * this rank owns.  scans are ALL sensors of the frame (every rank sees every
 * ray); each ray is traced only over the steps whose voxel lies in the rows
 * (y is monotone along a ray, so that is one step range, entered at its exact
 * walk state through the stateless keys of O5), and only returns in the rows
 * are binned.  The buffer map pushed holds the slab's voxels with LOCAL data
 * ranks (0..k_slab-1, in L order; the frame's global rank of a voxel = the k
 * of the slabs before + its local rank); voxels outside the rows are not
 * defined.  Every pass-through and return of the frame is counted by exactly
 * one rank, so the union of the slabs equals gvom_integrate_scan's map.  No
 * collective is needed for the map: the compute_maps_slab phases follow.
 * Not with GVOM_FLAG_PIPELINE or GVOM_FLAG_ROLLING.  With buffer_frames > 1
 * and motion a shifted older map reads rows of other slabs: set the peers
 * (gvom_set_peers).  Errors as gvom_integrate_scan, GVOM_E_INVALID for a bad
 * row range.                                                              */
GVOM_API gvom_status gvom_integrate_slab(gvom_handle* h, const gvom_scan* scans, int32_t n_scans,
                                         int32_t y0, int32_t y1);

/* The ray-segment partition with motion (buffer_frames > 1): a buffer map
 * shifted by the vehicle's motion reads rows that other ranks own.  With the
 * peers set, gvom_compute_maps_slab(phase 0) reads those rows -- LUT entries,
 * occupancy bits and data rows, at the same workspace offsets -- directly from
 * the owner's workspace (peer memory: each d_peer_workspaces[r] is rank r's
 * workspace as a pointer this GPU can load from, e.g. torch symmetric memory
 * buffer_ptrs of workspaces allocated there; d_peer_workspaces[rank] must be
 * this handle's own).  Every rank's handle has the same config (identical
 * layouts) and integrates every frame with gvom_integrate_slab over its slab
 * slab_y[rank]..slab_y[rank+1]; the caller orders a rank's reads after the
 * owners' integrate (a barrier) and the owners' next integrate after the
 * reads.  n_ranks = 0 clears.  The merged export (gvom_export_voxels) stays
 * local.                                                                  */
GVOM_API gvom_status gvom_set_peers(gvom_handle* h, const void* const* d_peer_workspaces,
                                    const int32_t* slab_y, int32_t n_ranks, int32_t rank);

/* Slab balancing for the ray-segment partition: d_out[y] (device, u64 [ny];
 * only [y0, y1) written) = the pass-throughs + returns of row y in the newest
 * buffer map, i.e. the sum over the row's voxels of misses + hits (P:105,
 * the counts the ray cast and the binning added).  A rank's ray-cast
 * work in its rows is proportional to it, so slab bounds that split the
 * summed rows evenly (parallel.balanced_slab_rows) even out the ranks.
 * Stream-ordered after the last integrate; not for rolling maps
 * (GVOM_E_INVALID); GVOM_E_EMPTY before the first integrate.              */
GVOM_API gvom_status gvom_row_work(gvom_handle* h, int32_t y0, int32_t y1, uint64_t* d_out);

/* Map processing: combine all buffer maps at the origin of the
 * newest one, then compute height, density, hard, soft, slope,
 * roughness and negative-obstacle layers.  GVOM_E_EMPTY if no map.         */
GVOM_API gvom_status gvom_compute_maps(gvom_handle* h);

/* Copy one layer of the last compute_maps into dst (host or device), which
 * must hold nx*ny*4 bytes (f32 layers) or nx*ny bytes (u8 layers), else
 * GVOM_E_SIZE.  Stream-ordered: synchronise before reading a host dst.     */
GVOM_API gvom_status gvom_export_2d(gvom_handle* h, gvom_layer layer, void* dst, size_t dst_bytes);

/* All layers at once ("each of these maps are published"):
 * dst[l] / dst_bytes[l] for l = GVOM_LAYER_HEIGHT..GVOM_LAYER_SPREAD, each
 * as in gvom_export_2d.  When every dst is 16-byte aligned device memory the
 * copy is one kernel launch; otherwise one async copy per layer.           */
GVOM_API gvom_status gvom_export_layers(gvom_handle* h, void* const dst[GVOM_LAYER_COUNT],
                                        const size_t dst_bytes[GVOM_LAYER_COUNT]);

/* One scan end to end: gvom_shift + gvom_integrate_scan + gvom_compute_maps
 * (+ gvom_export_layers when dst != NULL; + the costmap into cost_dst when
 * cost_weights != NULL, fused with the export as in gvom_export_layers_cost;
 * cost_weights and cost_dst are both NULL or both set), same arguments, results and
 * errors as those calls in sequence (inputs are validated before anything is
 * enqueued).  The frame's kernels are captured on the handle's stream and run
 * as ONE CUDA graph launch: the cached executable graph is patched with the
 * frame's arguments (cudaGraphExecUpdate) or re-instantiated when the launch
 * topology changed.  Falls back to plain stream launches (same kernels) when
 * capture does not apply: points or outputs in pageable host memory, or the
 * stream already under capture by the caller.  With GVOM_FLAG_PIPELINE the
 * step is two graphs -- integrate on the handle's stream, map processing and
 * export on the map stream -- whose slot fences are external event nodes, so
 * consecutive steps overlap; pinned host points are then copied on a
 * handle-owned copy stream into one of two staging buffers (overlapping the
 * previous scan's integrate), and pinned host outputs (without a costmap) are
 * exported into one of two device buffers and copied to the host on a second
 * copy stream (overlapping the next step's map processing): those host
 * outputs are complete after gvom_synchronize, not when the map stream
 * reaches the step.  The
 * graph and a private capture stream are driver objects held by the handle
 * (released by gvom_destroy); no device memory is allocated.              */
GVOM_API gvom_status gvom_step(gvom_handle* h, const double vehicle_xyz[3], const gvom_scan* scans,
                               int32_t n_scans, void* const dst[GVOM_LAYER_COUNT],
                               const size_t dst_bytes[GVOM_LAYER_COUNT],
                               const float cost_weights[7], void* cost_dst, size_t cost_bytes,
                               int64_t out_delta_voxels[3]);

/* gvom_step counters: out[0] graph launches, out[1] graph instantiations,
 * out[2] steps run without a graph.                                        */
GVOM_API gvom_status gvom_graph_stats(gvom_handle* h, int64_t out[3]);

/* Test hook (fault injection).  GVOM_FAULT_CAPTURE: the next gvom_step
 * capture fails as if cudaStreamEndCapture had failed; the step returns
 * GVOM_E_CUDA and the map state (buffer ring, slot origins, map-processing
 * bookkeeping) is rolled back to before the step's integrate, so the next
 * step continues as if the failed one had never been called (its shift
 * stands).  0 clears a pending fault.                                      */
#define GVOM_FAULT_CAPTURE 1
GVOM_API gvom_status gvom_debug_inject_fault(gvom_handle* h, int32_t what);

/* Costmap ("each of the output maps get some weight assigned to them
 * and the resulting per pixel sum is the cost in that pixel"; SURVEY 8(f)
 * NEXT-4).  cost = w0*hard + w1*soft + w2*density + w3*negative + w4*slope
 * + w5*roughness + w6*unknown, f32 in that order; a NaN layer contributes 0;
 * unknown = height undefined and not a negative obstacle (reading B5).
 * dst: nx*ny float32, host or device; ordered on the map stream.          */
GVOM_API gvom_status gvom_costmap(gvom_handle* h, const float weights[7], void* dst,
                                  size_t dst_bytes);

/* gvom_export_layers + gvom_costmap in ONE pass (NEXT-4 "fused into
 * export"): every layer cell is read once, written to dst[l] and folded into
 * the cost (same formula and order as gvom_costmap).  One kernel when every
 * destination is 4-byte aligned device memory; otherwise the two calls in
 * sequence.  Errors as those calls.                                        */
GVOM_API gvom_status gvom_export_layers_cost(gvom_handle* h, void* const dst[GVOM_LAYER_COUNT],
                                             const size_t dst_bytes[GVOM_LAYER_COUNT],
                                             const float weights[7], void* cost_dst,
                                             size_t cost_bytes);

/* GVOM_FLAG_ROLLING only: the window map, dense in L order over the current
 * window: hits, misses, m1, m2 (u64) and min_dz (u32, 0xFFFFFFFF where no
 * return) per voxel, each a caller-owned device array of nx*ny*nz entries.
 * GVOM_E_INVALID without the flag.  Stream-ordered.                       */
GVOM_API gvom_status gvom_export_window(gvom_handle* h, uint64_t* d_hits, uint64_t* d_misses,
                                        uint32_t* d_min_dz, uint64_t* d_m1, uint64_t* d_m2);

/* World-voxel origin of the last compute_maps (newest buffer map).  */
GVOM_API gvom_status gvom_map_origin(gvom_handle* h, int64_t out_origin[3]);

/* The combined voxel map of the last compute_maps encoded as in P:81:
 * d_lut[V] (rank in L order if occupied, else -1 - min(N_m, 2^30)) and
 * d_data[k] rows in L order.  Synchronous (reads k back).  Needs cap >= k
 * (else GVOM_E_SIZE with *out_k set).  The outputs P:297 calls "the
 * completed voxel map".                                                    */
GVOM_API gvom_status gvom_export_voxels(gvom_handle* h, int32_t* d_lut, gvom_voxel* d_data, int64_t cap,
                               int64_t* out_k);

/* One buffer map (age 0 = newest): its LUT, data rows and origin, as
 * produced by integrate_scan.  Synchronous.                               */
GVOM_API gvom_status gvom_export_frame(gvom_handle* h, int32_t age, int32_t* d_lut, gvom_voxel* d_data,
                              int64_t cap, int64_t* out_k, int64_t out_origin[3]);

/* ---- Multi-GPU slab partition -----------------------------
 * The points of one frame are sharded across P ranks (one process and handle
 * per GPU, not pipelined, not rolling); rank r owns the y-rows
 * [slab_y[r], slab_y[r+1]), which in L order is the contiguous voxel range
 * [slab_y[r]*nx*nz, slab_y[r+1]*nx*nz).  Per frame, with the collectives done
 * by the caller (torch.distributed / NCCL; paper_2109_13176_b200/parallel.py):
 *  1. gvom_partial_scan on the rank's sensors: a dense u32 miss grid [V] and
 *     the in-grid returns as gvom_endpoint records grouped by destination slab;
 *  2. reduce-scatter (SUM) of the miss grids by slab; all-to-all of records;
 *  3. gvom_slab_occupancy -> k of the slab; all-gather of k -> rank base
 *     (the k of the slabs before it) and the frame's total k;
 *  4. gvom_slab_finalize(base): LUT + data rows of the slab with GLOBAL ranks
 *     (data rows at [base, base + k) of the slot, so every rank's
 *     max_points_per_frame must cover the whole frame), pushed into the buffer;
 *  4b. with buffer_frames > 1 (motion: the shift of an older map reads rows of
 *     other slabs): all-gather the slabs' LUT rows and
 *     data rows into gvom_slot_buffers(age 0) of every rank, then
 *     gvom_slab_complete(total k): every rank holds the whole frame map;
 *  5. gvom_compute_maps_slab(phase 0): columns of the slab rows; all-gather of
 *     the q_s rows into gvom_surface_buffer() (and, with
 *     GVOM_FLAG_SLOPE_SKIP_OBSTACLES, of the hard / soft rows into
 *     gvom_obstacle_buffers()); phase 1: slope, roughness and negative
 *     obstacles of the slab rows [y0, y1) from the gathered surface (their
 *     windows and cones read the rows around the slab; with
 *     GVOM_FLAG_NEG_8CONE the 8-cone search still covers the whole map).
 *     Layers are defined on the slab rows only.
 * Sums and mins are exact integers, so the result is identical to one GPU.  */
typedef struct gvom_endpoint {
  uint32_t L;  /* linear voxel index of an in-grid return          */
  uint32_t dz; /* fixed-point height above the voxel floor (A12)   */
} gvom_endpoint;

GVOM_API gvom_status gvom_partial_scan(gvom_handle* h, const gvom_scan* scans, int32_t n_scans,
                                       uint32_t* d_miss, gvom_endpoint* d_ep, int64_t ep_cap,
                                       const int32_t* slab_y, int32_t n_ranks,
                                       int64_t* out_counts);
GVOM_API gvom_status gvom_slab_occupancy(gvom_handle* h, int32_t y0, int32_t y1,
                                         const gvom_endpoint* d_ep, int64_t n_ep, int64_t* out_k);
GVOM_API gvom_status gvom_slab_finalize(gvom_handle* h, int32_t y0, int32_t y1,
                                        const uint32_t* d_miss_slab, const gvom_endpoint* d_ep,
                                        int64_t n_ep, int64_t base);
/* NEXT-2 fused collective: steps 2 (the reduce-scatter of miss grids) and 4
 * in one kernel.  d_miss_grids: host array of the P ranks' partial miss grids
 * [V] (u32, 16-byte aligned) as device pointers this GPU can load from --
 * peer memory (e.g. torch symmetric memory buffer_ptrs, after a barrier that
 * orders the ranks' gvom_partial_scan before it); the finalize sums them over
 * the slab's tiles as it encodes them.  Same result as gvom_slab_finalize on
 * the reduce-scattered slab.  The grids must stay unchanged until the
 * handle's stream has passed this call.                                   */
GVOM_API gvom_status gvom_slab_finalize_peers(gvom_handle* h, int32_t y0, int32_t y1,
                                              const uint32_t* const* d_miss_grids,
                                              int32_t n_grids, const gvom_endpoint* d_ep,
                                              int64_t n_ep, int64_t base);
/* Device pointers of buffer map `age` (0 = newest): its LUT [nx*ny*nz] and
 * data rows [cap] (workspace memory; the caller writes the gathered slabs
 * into them, ordered on the handle's stream).                             */
GVOM_API gvom_status gvom_slot_buffers(gvom_handle* h, int32_t age, int32_t** out_d_lut,
                                       gvom_voxel** out_d_data, int64_t* out_cap);
/* After the all-gather of step 4b: rebuild the newest map's occupancy from its
 * complete LUT and set its occupied-voxel count to k_total.               */
GVOM_API gvom_status gvom_slab_complete(gvom_handle* h, int64_t k_total);
GVOM_API gvom_status gvom_compute_maps_slab(gvom_handle* h, int32_t y0, int32_t y1,
                                            int32_t phase);
/* the stream map processing is enqueued on (the handle's stream unless
 * GVOM_FLAG_PIPELINE): consumers of layers order themselves after it      */
GVOM_API gvom_status gvom_map_stream(gvom_handle* h, void** out_stream);
/* device pointer of the [ny][nx] int32 surface buffer (q_s, INT32_MIN = none) */
GVOM_API gvom_status gvom_surface_buffer(gvom_handle* h, int32_t** out_d_qs);
/* device pointers of the [ny][nx] u8 hard / soft layers: with
 * GVOM_FLAG_SLOPE_SKIP_OBSTACLES the slope windows of phase 1 read them across
 * slabs, so their rows are all-gathered along with the surface rows        */
GVOM_API gvom_status gvom_obstacle_buffers(gvom_handle* h, uint8_t** out_d_hard,
                                           uint8_t** out_d_soft);

/* Instrumentation.  gvom_set_timing(h, mask): every launch of a stage whose
 * bit (1 << GVOM_STAGE_*) is set in mask is bracketed by CUDA events on the
 * handle's stream (mask -1 = all stages, 0 = off); gvom_stage_times synchronises and
 * returns, per stage, [total ms, launches] pairs (2*GVOM_STAGE_COUNT
 * doubles), then clears the record.  gvom_launch_count returns the number of
 * kernels this handle has launched so far.                                  */
/* GVOM_STAGE_INTEGRATE / GVOM_STAGE_MAPS bracket a whole gvom_integrate_scan /
 * gvom_compute_maps call (one event pair around all its launches, recorded
 * inside gvom_step's graph too) instead of every launch.                   */
enum {
  GVOM_STAGE_RAYCAST = 0, GVOM_STAGE_RANK_COUNT, GVOM_STAGE_RANK_SCAN, GVOM_STAGE_FINALIZE,
  GVOM_STAGE_ENDPOINT, GVOM_STAGE_COLUMNS, GVOM_STAGE_SLOPE, GVOM_STAGE_NEGATIVE,
  GVOM_STAGE_MEMSET, GVOM_STAGE_H2D, GVOM_STAGE_EXPORT, GVOM_STAGE_MERGE,
  GVOM_STAGE_INTEGRATE, GVOM_STAGE_MAPS, GVOM_STAGE_COUNT
};
GVOM_API gvom_status gvom_set_timing(gvom_handle* h, int32_t enable);
GVOM_API gvom_status gvom_stage_times(gvom_handle* h, double* out, int32_t n_doubles);
GVOM_API int64_t gvom_launch_count(const gvom_handle* h);

GVOM_API const char* gvom_status_string(gvom_status s);
GVOM_API int32_t gvom_abi_version(void);

#ifdef __cplusplus
}
#endif
#endif /* GVOM_H */
