// gvom_device.cuh -- device helpers shared by the kernels (one copy of every
// rule that decides an integer bit-exactly: the transform of O3).
// Independent of oracle/ (no shared code, headers or tables).
#pragma once

#include "gvom_internal.cuh"

namespace gvom {

constexpr float kGLim = 4194304.0f;  // |g_i| < 2^22 voxels (reading A5)

// O3: g_i = ((A_i0 x + A_i1 y) + A_i2 z) + b_i, f32 RN each, no
// contraction (explicit _rn intrinsics; the library is built -fmad=false).
// Valid iff finite, not the (0,0,0) no-return, and every |g_i| < 2^22 (A5).
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

// inclusive warp scan (Hillis-Steele over shuffles)
__device__ __forceinline__ uint32_t warp_incl_scan(uint32_t v, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

}  // namespace gvom
