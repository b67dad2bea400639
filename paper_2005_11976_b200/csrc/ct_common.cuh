// ct_common.cuh -- shared device helpers, geometry policies and argument
// checks of the cone-beam FP / BP / SART kernels (see ct_fp.cu, ct_bp.cu,
// ct_sample.cu, ct_pose.cu; include/cyltomo_b200.h for the C-ABI).
//
//
// Reference semantics restated (not translated) from
//   /root/reference/pkg/src/cyltomo/_kernels.py  (forward_cyl :238-293,
//   forward_cart :296-343, backproject_cyl :380-417, backproject_cart
//   :420-443, interp_* :48-151, intervals :170-231)
//   /root/reference/pkg/src/cyltomo/recon.py     (correction / update :88-120,
//   residual :148-153)
//
// Numerics:
//  * per-ray setup -- sub-ray direction, support interval, sample count
//    n = ceil((t1-t0)/step) and the in-support test of the last sample -- is
//    done in fp64 with explicitly rounded ops (no FMA contraction), i.e. the
//    same IEEE operation sequence as the reference, so sample counts and the
//    SART row sums w are bit-identical to the fp64 oracle;
//  * the march itself is fp32, relative to the first sample position, with
//    the support convexity argument: samples 0..n-2 lie inside the support
//    by >= step/2 along the ray, only sample n-1 can fall outside;
//  * BP computes (u,v) in fp32 and recomputes them in fp64 (reference
//    arithmetic) only when a footprint lies within 1e-3 px of the detector
//    frame edge, where the `den > 0` decision is discontinuous.
#pragma once
#include "cyltomo_b200.h"

#include <cuda_runtime.h>
#include <cassert>
#include <limits.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define CT_STREAM(s) (static_cast<cudaStream_t>(s))

// error state of the C-ABI (ct_abi.cu)
namespace ctabi {
extern thread_local char g_err[512];
int set_err(int code, const char* msg);
int check_launch(const char* what);
}  // namespace ctabi

namespace {
using ctabi::check_launch;
using ctabi::g_err;
using ctabi::set_err;

#ifndef CT_ATAN_TERMS
#define CT_ATAN_TERMS 7          // 2 atan polynomial terms (7: 4.8e-7 rad; 8: 5.7e-8 rad)
#endif
constexpr double kPi = 3.141592653589793;
constexpr double kTwoPi = 2.0 * kPi;
constexpr float kTwoPiF = 6.28318530717958647692f;


// ---------------------------------------------------------------------------
// exact fp64 helpers: the reference evaluates a*b+c as two rounded ops
// ---------------------------------------------------------------------------
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }
__device__ __forceinline__ double dsqrt(double a) { return __dsqrt_rn(a); }

// Unit direction of the sub-ray through detector point (cu, cv)
// (_kernels.py:263-272): ((o + cu*du) + cv*dv) - src, normalised.
__device__ __forceinline__ void subray_dir(const ct_ray_view& v, double cu, double cv,
                                           double d[3]) {
  double dx = dsub(dadd(dadd(v.origin[0], dmul(cu, v.du[0])), dmul(cv, v.dv[0])), v.src[0]);
  double dy = dsub(dadd(dadd(v.origin[1], dmul(cu, v.du[1])), dmul(cv, v.dv[1])), v.src[1]);
  double dz = dsub(dadd(dadd(v.origin[2], dmul(cu, v.du[2])), dmul(cv, v.dv[2])), v.src[2]);
  double norm = dsqrt(dadd(dadd(dmul(dx, dx), dmul(dy, dy)), dmul(dz, dz)));
  d[0] = ddiv(dx, norm);
  d[1] = ddiv(dy, norm);
  d[2] = ddiv(dz, norm);
}


// ---------------------------------------------------------------------------
// fp32 sampling helpers (no XU-pipe conversions on the hot loop)
// ---------------------------------------------------------------------------
// floor(x) for 0 <= x < 2^22 on the FMA pipe: x + 2^23 rounded toward -inf is
// floor(x) + 2^23 exactly; its bit pattern minus 0x4B000000 is the integer.
__device__ __forceinline__ float floor_pos(float x, int& i) {
  const float t = __fadd_rd(x, 8388608.0f);
  i = __float_as_int(t) - 0x4B000000;
  return t - 8388608.0f;
}


__device__ __forceinline__ float sqrt_approx(float x) {
  float r;
  asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// theta = atan2(y, x) mapped to [0, 2pi) as the reference does (_kernels.py:287-289):
// octant reduction + a degree-13 odd minimax polynomial (|err| < 3.3e-7 rad in
// fp32, i.e. < 6e-5 of a theta cell at n_theta = 1024 -- the same size as the
// fp32 resolution of the theta index itself).
__device__ __forceinline__ float theta_2pi(float y, float x) {
  const float ax = fabsf(x), ay = fabsf(y);
  const float mx = fmaxf(ax, ay), mn = fminf(ax, ay);
  float rc;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rc) : "f"(fmaxf(mx, 1e-30f)));
  const float a = mn * rc;   // in [0, 1]; 0 on the axis (atan2(0, 0) = 0)
  const float s = a * a;
  float p = 0.0068140108452664225f;
  p = fmaf(p, s, -0.033610868703448114f);
  p = fmaf(p, s, 0.07963126616806604f);
  p = fmaf(p, s, -0.13233753525313302f);
  p = fmaf(p, s, 0.19807922265216282f);
  p = fmaf(p, s, -0.3331737967047227f);
  p = fmaf(p, s, 0.999996115058577f);
  float t = a * p;
  t = (ay > ax) ? (1.57079632679489662f - t) : t;
  t = (x < 0.0f) ? (3.14159265358979324f - t) : t;
  return (y < 0.0f) ? (kTwoPiF - t) : t;
}

// Trilinear interpolation as a polynomial in the cell weights:
//   f = c0 + cr wr + ct wt + ch wh + crt wr wt + crh wr wh + cth wt wh + crth wr wt wh
// from the 8 corner values a = (k0,j0,i0) (k0,j0,i1) (k0,j1,i0) (k0,j1,i1), b = the
// same at k1.  The gather layout stores the coefficients (same 32 bytes as the
// values), so a sample is 7 dependent-depth-3 FFMAs and no FADD; the plain
// path derives them in-kernel with the same fp32 ops, so both paths give
// identical bits.
__device__ __forceinline__ void trilinear_coeffs(float4 a, float4 b, float4& ca, float4& cb) {
  const float dr0 = a.y - a.x, dr1 = a.w - a.z, dr2 = b.y - b.x, dr3 = b.w - b.z;
  const float dt0 = a.z - a.x, dt1 = b.z - b.x;
  ca = make_float4(a.x, dr0, dt0, dr1 - dr0);                        // c0, cr, ct, crt
  cb = make_float4(b.x - a.x, dr2 - dr0, dt1 - dt0, (dr3 - dr2) - (dr1 - dr0));  // ch, crh, cth, crth
}
__device__ __forceinline__ float trilinear_eval_scalar(float4 ca, float4 cb, float wr, float wt,
                                                      float wh) {
  const float e1 = fmaf(cb.w, wh, ca.w);   // crt + crth wh
  const float e0 = fmaf(cb.y, wh, ca.y);   // cr + crh wh
  const float f1 = fmaf(cb.z, wh, ca.z);   // ct + cth wh
  const float f0 = fmaf(cb.x, wh, ca.x);   // c0 + ch wh
  return fmaf(fmaf(e1, wt, e0), wr, fmaf(f1, wt, f0));
}

// one bilinear footprint (ct_pack_quads) with a single 128-bit load
__device__ __forceinline__ float4 ld_quad(const float4* p) {
  float4 q;
#if defined(CT_QUAD_LOAD_NOALLOC)
  asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w) : "l"(p));
#else
  asm("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w) : "l"(p));
#endif
  return q;
}

// one corner quad of the large-volume layout (GL_QUAD)
// (L1-allocating: in the large volumes neighbouring rays do meet in L1; A/B
// at C5 -19 % against no_allocate)
__device__ __forceinline__ float4 ld_vquad(const float4* p) {
  float4 q;
  asm("ld.global.nc.v4.f32 {%0,%1,%2,%3}, [%4];"
      : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w) : "l"(p));
  return q;
}

// one 32-byte cell of the gather layout with a single 256-bit load
// (sm_100 LDG.E.NA.ENL2.256; read-only path).  L1::no_allocate: the cells of
// one ray are reused in registers and neighbouring rays rarely meet in L1, so
// allocating L1 lines only costs data-pipe fill wavefronts (A/B: -5.5% FP time)
__device__ __forceinline__ void ld_cell(const float4* p, float4& a, float4& b) {
#if defined(CT_CELL_LOAD_ALLOC)
  asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
                 "=f"(b.w)
               : "l"(p));
#else
  asm("ld.global.nc.L1::no_allocate.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z),
                 "=f"(b.w)
               : "l"(p));
#endif
}


// ---------------------------------------------------------------------------
// packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2): two samples per
// instruction for the per-sample coordinate / index / weight math.  Each lane
// of an f32x2 op is the IEEE op of the scalar code, and both the gather and
// the plain path use the same paired code for the same samples, so their
// results are bit-identical.
// ---------------------------------------------------------------------------
typedef unsigned long long f32x2;

__device__ __forceinline__ f32x2 pk(float a, float b) {
  f32x2 r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(f32x2 v, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(v));
}
__device__ __forceinline__ f32x2 fma2(f32x2 a, f32x2 b, f32x2 c) {
  f32x2 d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ f32x2 mul2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 sub2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 add2_rd(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("add.rm.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ f32x2 dup2(float a) { return pk(a, a); }
__device__ __forceinline__ uint2 bits2(f32x2 v) {
  uint2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=r"(r.x), "=r"(r.y) : "l"(v));
  return r;
}
__device__ __forceinline__ f32x2 add2(f32x2 a, f32x2 b) {
  f32x2 d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// The same 7 FMAs as trilinear_eval_scalar, lane for lane, in 4 issue slots:
// the 32-byte cell lands in 8 consecutive registers, so (c0, cr), (ct, crt),
// (ch, crh), (cth, crth) are register pairs and the h and theta steps run as
// FFMA2 with the weight broadcast: (f0, e0) = (ch, crh) wh + (c0, cr),
// (f1, e1) = (cth, crth) wh + (ct, crt), (F, E) = (f1, e1) wt + (f0, e0),
// f = E wr + F.
__device__ __forceinline__ float trilinear_eval(float4 ca, float4 cb, float wr, float wt, float wh) {
#if defined(CT_EVAL_SCALAR)
  return trilinear_eval_scalar(ca, cb, wr, wt, wh);
#else
  const f32x2 WH = dup2(wh);
  const f32x2 FE0 = fma2(pk(cb.x, cb.y), WH, pk(ca.x, ca.y));
  const f32x2 FE1 = fma2(pk(cb.z, cb.w), WH, pk(ca.z, ca.w));
  float F, E;
  upk(fma2(FE1, dup2(wt), FE0), F, E);
  return fmaf(E, wr, F);
#endif
}

// 2 atan(q) / q as a polynomial in q^2 on q in [-1, 1] (odd minimax fits of
// 2 atan, tools/fit_atan.py)
#if CT_ATAN_TERMS == 6
// degree-11 fit (3.3e-6 rad; A/B only)
#define CT_ATAN2X_C7 0.0f
#define CT_ATAN2X_C6 0.0f
#define CT_ATAN2X_C5 -0.023422138765454292f
#define CT_ATAN2X_C4 0.10525291413068771f
#define CT_ATAN2X_C3 -0.23281531035900116f
#define CT_ATAN2X_C2 0.38706788420677185f
#define CT_ATAN2X_C1 -0.665244996547699f
#define CT_ATAN2X_C0 1.9999547004699707f
#elif CT_ATAN_TERMS == 7
// degree-13 odd minimax fit (4.8e-7 rad, 6.3e-7 evaluated in fp32 -- about
// one fp32 ulp of theta near 2 pi; FP parity margins are unchanged, see
// tools/parity_margins.py)
#define CT_ATAN2X_C7 0.0f
#define CT_ATAN2X_C6 0.013589471578598022f
#define CT_ATAN2X_C5 -0.06711680442094803f
#define CT_ATAN2X_C4 0.15916450321674347f
#define CT_ATAN2X_C3 -0.26464372873306274f
#define CT_ATAN2X_C2 0.3961613178253174f
#define CT_ATAN2X_C1 -0.6663504242897034f
#define CT_ATAN2X_C0 1.9999924898147583f
#else
#define CT_ATAN2X_C7 -0.008428506553173065f
#define CT_ATAN2X_C6 0.044908907264471054f
#define CT_ATAN2X_C5 -0.1135723665356636f
#define CT_ATAN2X_C4 0.1941567361354828f
#define CT_ATAN2X_C3 -0.2787010073661804f
#define CT_ATAN2X_C2 0.3990408182144165f
#define CT_ATAN2X_C1 -0.6666072607040405f
#define CT_ATAN2X_C0 1.999998927116394f
#endif
constexpr double kAtan2x[8] = {CT_ATAN2X_C0, CT_ATAN2X_C1, CT_ATAN2X_C2, CT_ATAN2X_C3,
                               CT_ATAN2X_C4, CT_ATAN2X_C5, CT_ATAN2X_C6, CT_ATAN2X_C7};
// The polynomial with coefficients pre-scaled by 1/dtheta (CylGeo::tc): the
// theta index is then one FFMA away, fma(q, p(q^2), ct).
__device__ __forceinline__ float atan2x_poly(const float* c, float s) {
  float p = CT_ATAN_TERMS == 6 ? c[5] : CT_ATAN_TERMS == 7 ? c[6] : fmaf(c[7], s, c[6]);
#pragma unroll
  for (int i = CT_ATAN_TERMS == 6 ? 4 : 5; i >= 0; --i) p = fmaf(p, s, c[i]);
  return p;
}
__device__ __forceinline__ f32x2 atan2x_poly2(const float* c, f32x2 s) {
  f32x2 p = CT_ATAN_TERMS == 6 ? dup2(c[5])
           : CT_ATAN_TERMS == 7 ? dup2(c[6]) : fma2(dup2(c[7]), s, dup2(c[6]));
#pragma unroll
  for (int i = CT_ATAN_TERMS == 6 ? 4 : 5; i >= 0; --i) p = fma2(p, s, dup2(c[i]));
  return p;
}

// Per-ray march constants.  Sample k of a ray sits at e + k*i (grid frame).
//  * Cartesian: (ex, ey, ez) + k*(ix, iy, iz), in index units folded by locate.
//  * Cylindrical: the ray's trace in the (x, y) plane is a line at distance
//    d0 from the axis; with s the signed distance along it from the foot of
//    the perpendicular, oriented so that theta increases with s,
//        r = sqrt(s^2 + d0^2),   theta = phi + 2 atan(s / (r + d0))
//    (half-angle form: |s / (r + d0)| <= 1, so no octant reduction), where
//    phi is the foot's angle, shifted by 2 pi so the ray's smallest theta lies
//    in [0, 2 pi).  s and d0 are in r-index units, the h index is linear in k:
//        s = es + k*is,   h index + 1 = eh + k*ih,
//    and ct = phi / dtheta + 0.5 folds the theta index offset (+1 halo, -0.5
//    cell centre).  A ray spans < pi in theta; one that crosses theta = 2 pi
//    (wrap) has its rows past n_theta wrapped in the integer cell index
//    (CylGeo::gather_index<true>), taken warp-uniformly by march().
struct RayF {
  float ex, ey, ez, ix, iy, iz;   // Cartesian, and the cylindrical nearest mode
  float es, is, eh, ih, d0, d2, ct;
  bool wrap;                      // cylindrical: the ray's theta index passes n_theta
};

// One sample's trilinear cell: bit patterns of floor(index + 1) (+0x4B000000,
// the "+1" being the gather layout's halo offset; the cylindrical r bits carry
// one less, see kRMagic) and the three weights.
struct Cell {
  unsigned ib, jb, kb;
  float w0, w1, w2;
};

constexpr unsigned kMagicBits = 0x4B000000u;   // bits of 2^23
// r floor: x + (2^23 - 1/2) rounded toward -inf has the bits of
// 2^23 + floor(x + 1/2) - 1 (for x < 1/2 the grid below 2^23 still gives bits
// 2^23 - 1), and x - (that - (2^23 - 1/2)) is frac(x + 1/2) exactly: the
// cell-centre offset costs no add.  (For x < 1/2 -- the axis half-cell -- the
// weight is off, but that cell is the r halo whose r terms are zero.)
constexpr float kRMagic = 8388607.5f;

// ---------------------------------------------------------------------------
// grid policies: support interval (fp64), last-sample test (fp64) and the
// fp32 trilinear sample
// ---------------------------------------------------------------------------
// Gather-layout strides in cells: r (x) fastest, row stride js = n + 1, layer
// stride ks = rows * js padded so that ks + js + 1 == 0 (mod 256).  The floor
// bit patterns carry the magic 2^23 = 75 * 2^24 (bits B = 0x4B000000), so
// B * (ks + js + 1) == 0 (mod 2^32) and kb*ks + jb*js + ib is the cell index
// itself: no bias term per sample.
__host__ __device__ inline unsigned gather_layer_stride(unsigned rows, unsigned js) {
  const unsigned ks = rows * js;
  return ks + (256u - (ks + js + 1u) % 256u) % 256u;
}

struct CellStrides {
  unsigned js, ks;
};
// gather-layout base pointer for gather_index's cell numbers: `one_on` cells
// on (the cylindrical r floor bits carry index - 1)
__host__ inline const float4* cell_base(const float* gather, bool quad, int one_on) {
  return reinterpret_cast<const float4*>(gather) + (quad ? 1 : 2) * one_on;
}
// signed cell offset of a gather_index value (the first cylindrical cell is -1)
__device__ __forceinline__ ptrdiff_t cell_off(unsigned idx) { return (ptrdiff_t)(int)idx; }
// CT_QUAD_BRICK: GL_QUAD cells stored in 2x2x2 (layer, row, column) bricks,
// one 128-byte line each: the two layers of a trilinear cell share a line for
// even layers, and neighbouring rays' cells share lines in theta as well as r
// (A/B: C5 0.298 -> 0.265 s per object-iteration, C4-cyl FP 0.508 -> 0.453 s).
#ifndef CT_QUAD_BRICK
#define CT_QUAD_BRICK 1
#endif
#ifndef CT_QB_LK
#define CT_QB_LK 1               // log2 layers per GL_QUAD brick
#endif
#ifndef CT_QB_LJ
#define CT_QB_LJ 1               // log2 rows per GL_QUAD brick (columns: the rest of 8 cells)
#endif
constexpr unsigned QB_LK = CT_QB_LK, QB_LJ = CT_QB_LJ, QB_LI = 3 - CT_QB_LK - CT_QB_LJ;
__host__ __device__ inline unsigned qbricks(unsigned n, unsigned l) { return (n + (1u << l) - 1u) >> l; }
__host__ __device__ __forceinline__ unsigned quad_brick_index(unsigned kc, unsigned jc,
                                                              unsigned ic, unsigned jbr,
                                                              unsigned ibr) {
  return ((((kc >> QB_LK) * jbr + (jc >> QB_LJ)) * ibr + (ic >> QB_LI)) << 3) |
         ((kc & ((1u << QB_LK) - 1u)) << (QB_LJ + QB_LI)) |
         ((jc & ((1u << QB_LJ) - 1u)) << QB_LI) | (ic & ((1u << QB_LI) - 1u));
}
// The bricked GL_QUAD cell of layer kc + 1 from that of layer kc: the next
// slot of the brick, or (last layer of a brick) the first layer slot of the
// next brick layer, brick_layer = cells per brick layer (jbr * ibr * 8).
// Same value as quad_brick_index(kc + 1, jc, ic, ...), fewer integer ops.
__host__ __device__ __forceinline__ unsigned quad_next_layer(unsigned idx, unsigned kc,
                                                             unsigned brick_layer) {
  constexpr unsigned kmask = (1u << QB_LK) - 1u, kstep = 1u << (QB_LJ + QB_LI);
  return (kc & kmask) == kmask ? idx - kmask * kstep + brick_layer : idx + kstep;
}
// GL_OCTB: GL_OCT cells in 2x2 (row, column) bricks per layer, one 128-byte
// line each (gather_obrick)
__host__ __device__ __forceinline__ unsigned oct_brick_index(unsigned kc, unsigned jc,
                                                             unsigned ic, unsigned jbr,
                                                             unsigned ibr) {
  return (((kc * jbr + (jc >> 1)) * ibr + (ic >> 1)) << 2) | ((jc & 1u) << 1) | (ic & 1u);
}
// rows x ncols real cells per layer
__host__ __device__ inline CellStrides cell_strides(unsigned rows, unsigned ncols) {
  CellStrides c;
  c.js = ncols;
  c.ks = gather_layer_stride(rows, ncols);
  return c;
}

// Large volumes use 16-byte per-layer bilinear cells (GL_QUAD) instead of the
// 32-byte trilinear cells: half the bytes per h layer, so more of the band of
// layers a wave of rays works on stays in L2, for one more load and two f32x2
// subtractions per cell entered.  Measured (A/B): C5 -23.5 %, C4-cyl equal,
// C4-cart (8.4 MB layers) +22 %, C2 (4.2 MB layers) +15 %; hence layers above
// 10 MB.  CT_GATHER_QUAD=0/1 overrides.
inline bool gather_quad(double cells_per_layer) {
  const char* e = getenv("CT_GATHER_QUAD");
  if (e && *e) return e[0] == '1';
  return 32.0 * cells_per_layer > 10.0e6;
}
// 32-byte cells in 2x2 bricks (GL_OCTB) when the layers exceed the
// small-layer bound of the FP (CT_FP_SMALL_LAYER_BYTES; A/B: C4-cart -6 %,
// C2 +15 %).  CT_GATHER_OBRICK=0/1 overrides.
#ifndef CT_FP_SMALL_LAYER_BYTES
#define CT_FP_SMALL_LAYER_BYTES 6.0e6
#endif
inline bool gather_obrick(double cells_per_layer) {
  if (gather_quad(cells_per_layer)) return false;
  const char* e = getenv("CT_GATHER_OBRICK");
  if (e && *e) return e[0] == '1';
  return 32.0 * cells_per_layer > CT_FP_SMALL_LAYER_BYTES;
}

struct CylGeo {
  const float* __restrict__ mu;
  const float4* __restrict__ oct;  // gather layout (ct_pack_gather_cyl) or null
  bool quad;                       // oct holds GL_QUAD corner quads
  bool obrick;                     // oct holds GL_OCTB bricked 32-byte cells
  long long dbg_floats = 0;        // CT_DEBUG_BOUNDS: gather buffer length (floats)
  int nh, nt, nr;
  double radius, half_h;
  // fp32 sampling constants
  float inv_dr, inv_dth, inv_dh, h_off, h_off1, nr_m1, nh_m1;
  float tc[8];   // 2 atan polynomial coefficients times n_theta / (2 pi)
  // gather layout: cells (nh+1, nt+1, nr+1), strides (ks, js, 1)
  unsigned cell_kstride, cell_jstride, jb_wrap;
  double cells_layer;   // real cells per layer (rows x columns)
  const float4* __restrict__ qraw;   // GL_QUAD bricked layout (CT_QUAD_BRICK)
  unsigned long long qtex = 0;       // CT_QUAD_TEX: texture object over qraw (A/B)
  unsigned brick_j, brick_i;         // GL_OCTB bricks per layer: rows / 2, columns / 2
  unsigned qbrick_j, qbrick_i;       // GL_QUAD bricks per layer pair
  unsigned qbrick_layer;             // GL_QUAD cells per brick layer (qbrick_j * qbrick_i * 8)

  __host__ void init(const float* m, const float* gather, const ct_cyl_grid& g) {
    mu = m;
    nh = g.n_h; nt = g.n_theta; nr = g.n_r;
    radius = g.radius;
    half_h = 0.5 * g.height;
    inv_dr = (float)(g.n_r / g.radius);
    inv_dth = (float)(g.n_theta / kTwoPi);
    for (int i = 0; i < 8; ++i) tc[i] = (float)(kAtan2x[i] * (g.n_theta / kTwoPi));
    inv_dh = (float)(g.n_h / g.height);
    h_off = (float)(0.5 * g.n_h - 0.5);
    nr_m1 = (float)(g.n_r - 1);
    nh_m1 = (float)(g.n_h - 1);
    h_off1 = h_off + 1.0f;
    const unsigned B = kMagicBits;
    const CellStrides cs = cell_strides((unsigned)gather_rows(g.n_theta), (unsigned)g.n_r + 1u);
    cell_jstride = cs.js;
    cell_kstride = cs.ks;
    cells_layer = (double)gather_rows(g.n_theta) * (g.n_r + 1);
    quad = gather_quad(cells_layer);
    obrick = gather_obrick(cells_layer);
    // the r floor bits carry index - 1 (kRMagic): the base is one cell on
    oct = gather ? cell_base(gather, quad, 1) : nullptr;
    qraw = reinterpret_cast<const float4*>(gather);
    brick_j = ((unsigned)gather_rows(g.n_theta) + 1u) / 2u;
    brick_i = ((unsigned)g.n_r + 2u) / 2u;
    qbrick_j = qbricks((unsigned)gather_rows(g.n_theta), QB_LJ);
    qbrick_i = qbricks((unsigned)g.n_r + 1u, QB_LI);
    qbrick_layer = qbrick_j * qbrick_i * 8u;
    jb_wrap = B + (unsigned)g.n_theta;
  }
  // theta rows of the gather layout: indices -1 .. n_theta - 1 (see RayF)
  __host__ __device__ static int gather_rows(int n_theta) { return n_theta + 1; }

  // _kernels.py:170-204 (same operation order)
  __device__ __forceinline__ bool interval(const double s[3], const double d[3], double& t0,
                                           double& t1) const {
    double tr0, tr1, tz0, tz1;
    double a = dadd(dmul(d[0], d[0]), dmul(d[1], d[1]));
    if (a < 1e-18) {
      if (dadd(dmul(s[0], s[0]), dmul(s[1], s[1])) > dmul(radius, radius)) return false;
      tr0 = -1e30; tr1 = 1e30;
    } else {
      double b = dadd(dmul(s[0], d[0]), dmul(s[1], d[1]));
      double c = dsub(dadd(dmul(s[0], s[0]), dmul(s[1], s[1])), dmul(radius, radius));
      double disc = dsub(dmul(b, b), dmul(a, c));
      if (disc <= 0.0) return false;
      double sq = dsqrt(disc);
      tr0 = ddiv(dsub(-b, sq), a);
      tr1 = ddiv(dadd(-b, sq), a);
    }
    if (fabs(d[2]) < 1e-18) {
      if (fabs(s[2]) > half_h) return false;
      tz0 = -1e30; tz1 = 1e30;
    } else {
      tz0 = ddiv(dsub(-half_h, s[2]), d[2]);
      tz1 = ddiv(dsub(half_h, s[2]), d[2]);
      if (tz0 > tz1) { double tmp = tz0; tz0 = tz1; tz1 = tmp; }
    }
    t0 = fmax(fmax(tr0, tz0), 0.0);
    t1 = fmin(tr1, tz1);
    return true;
  }

  // in-support test of a sample at parameter t (_kernels.py:280-286)
  __device__ __forceinline__ bool inside(const double s[3], const double d[3], double t) const {
    double x = dadd(s[0], dmul(t, d[0]));
    double y = dadd(s[1], dmul(t, d[1]));
    double z = dadd(s[2], dmul(t, d[2]));
    double r = dsqrt(dadd(dmul(x, x), dmul(y, y)));
    return !(r > radius || z < -half_h || z > half_h);
  }
  // the interpolator's own zero-outside test (_kernels.py:56-57) is the same
  // expression as `inside` for cylinders
  __device__ __forceinline__ bool interp_nonzero(const double*, const double*, double) const {
    return true;
  }

  // Per-ray constants (RayF) from the first sample position e and the step
  // vector inc (grid frame, fp64); samples 0..n-1.
  __device__ __forceinline__ void setup_ray(const double e[3], const double inc[3], int n,
                                            RayF& ry) const {
    ry.ex = (float)e[0]; ry.ey = (float)e[1]; ry.ez = (float)e[2];
    ry.ix = (float)inc[0]; ry.iy = (float)inc[1]; ry.iz = (float)inc[2];
    const double l2 = inc[0] * inc[0] + inc[1] * inc[1];
    double es, is, d0, phi;
    if (l2 > 0.0) {
      const double l = sqrt(l2), ux = inc[0] / l, uy = inc[1] / l;
      const double c = e[0] * uy - e[1] * ux;        // > 0: theta increases along the ray
      const double sg = c >= 0.0 ? 1.0 : -1.0;
      d0 = fabs(c);
      es = sg * (e[0] * ux + e[1] * uy);
      is = sg * l;
      phi = atan2(uy, ux) - sg * (0.5 * kPi);         // angle of the foot point
    } else {                                          // parallel to the axis
      es = 0.0; is = 0.0;
      d0 = sqrt(e[0] * e[0] + e[1] * e[1]);
      phi = atan2(e[1], e[0]);
    }
    // shift phi by 2 pi so the smallest theta of samples 0..n-1 is in [0, 2 pi)
    // The 2 pi shift and the wrap flag only need the ray's theta range to
    // ~1e-4 rad: fp32 atan2 (a few ulp) with margins.  Shifted so theta >=
    // -2e-4 (the theta index stays >= 0.5 - 2e-4 n_theta / 2 pi > 0); wrap set
    // whenever the range may reach 2 pi (the wrap loop is always correct).
    const double s_last = es + (n - 1) * is;
    const float d0f = (float)d0;
    const double th_min = phi + (double)atan2f((float)fmin(es, s_last), d0f);
    phi -= kTwoPi * floor((th_min + 1e-4) / kTwoPi);
    const double th_max = phi + (double)atan2f((float)fmax(es, s_last), d0f);
    ry.wrap = th_max + 1e-4 >= kTwoPi * (1.0 - 1e-3 / nt);
    const double idr = (double)nr / radius, d0i = fmax(d0 * idr, 1e-30);
    ry.es = (float)(es * idr);
    ry.is = (float)(is * idr);
    ry.d0 = (float)d0i;
    ry.d2 = (float)(d0i * d0i);
    ry.ct = (float)(phi * ((double)nt / kTwoPi) + 0.5);
    ry.eh = (float)(e[2] * ((double)nh / (2.0 * half_h)) + (0.5 * nh + 0.5));
    ry.ih = (float)(inc[2] * ((double)nh / (2.0 * half_h)));
  }

  // Trilinear cell of sample k (see RayF): r = sqrt(s^2 + d0^2) and
  // theta = phi + 2 atan(s / (r + d0)) with 2 atan from a degree-13 odd
  // minimax polynomial on [-1, 1] (4.8e-7 rad; 6.3e-7 evaluated in fp32).
  // floor() via x + 2^23 rounded toward -inf (bits = floor(x) + 0x4B000000).
  // The indices carry the gather layout's +1 halo offset.
  __device__ __forceinline__ Cell locate1(float k, const RayF& ry) const {
    const float s = fmaf(k, ry.is, ry.es);
    const float fh1 = fmaf(k, ry.ih, ry.eh);
    const float r = sqrt_approx(fmaf(s, s, ry.d2));
    const float q = __fmul_rn(s, rcp_approx(__fadd_rn(r, ry.d0)));
    const float ft1 = fmaf(q, atan2x_poly(tc, __fmul_rn(q, q)), ry.ct);
    const float tr = __fadd_rd(r, kRMagic);
    const float th_ = __fadd_rd(fh1, 8388608.0f);
    const float tt = __fadd_rd(ft1, 8388608.0f);
    Cell c;
    c.w0 = __fsub_rn(r, __fsub_rn(tr, kRMagic));
    c.w1 = __fsub_rn(ft1, __fsub_rn(tt, 8388608.0f));
    c.w2 = __fsub_rn(fh1, __fsub_rn(th_, 8388608.0f));
    c.ib = __float_as_uint(tr);
    c.jb = __float_as_uint(tt);
    c.kb = __float_as_uint(th_);
    return c;
  }

  // the same for samples ka, kb, two per f32x2 instruction (lane-for-lane
  // the ops of locate1, so both give identical bits)
  __device__ __forceinline__ void locate2(f32x2 K, const RayF& ry, Cell& ca, Cell& cb) const {
    const f32x2 S = fma2(K, dup2(ry.is), dup2(ry.es));
    const f32x2 FH1 = fma2(K, dup2(ry.ih), dup2(ry.eh));
    float r2a, r2b;
    upk(fma2(S, S, dup2(ry.d2)), r2a, r2b);
    const f32x2 R = pk(sqrt_approx(r2a), sqrt_approx(r2b));
    float rda, rdb;
    upk(add2(R, dup2(ry.d0)), rda, rdb);
    const f32x2 Q = mul2(S, pk(rcp_approx(rda), rcp_approx(rdb)));
    const f32x2 FT1 = fma2(Q, atan2x_poly2(tc, mul2(Q, Q)), dup2(ry.ct));

    const f32x2 BIG = dup2(8388608.0f);
    const f32x2 RM = dup2(kRMagic);
    const f32x2 TR = add2_rd(R, RM), TT = add2_rd(FT1, BIG), TH = add2_rd(FH1, BIG);
    const f32x2 WR = sub2(R, sub2(TR, RM)), WT = sub2(FT1, sub2(TT, BIG));
    const f32x2 WH = sub2(FH1, sub2(TH, BIG));
    upk(WR, ca.w0, cb.w0);
    upk(WT, ca.w1, cb.w1);
    upk(WH, ca.w2, cb.w2);
    float t0, t1;
    upk(TR, t0, t1);
    ca.ib = __float_as_uint(t0); cb.ib = __float_as_uint(t1);
    upk(TT, t0, t1);
    ca.jb = __float_as_uint(t0); cb.jb = __float_as_uint(t1);
    upk(TH, t0, t1);
    ca.kb = __float_as_uint(t0); cb.kb = __float_as_uint(t1);
  }

  // gather-layout cell index (modular uint32; one constant for all offsets)
  template <bool WRAP>
  __device__ __forceinline__ unsigned gather_index(const Cell& c) const {
    // WRAP (rays crossing theta = 2 pi): rows past n_theta wrap onto the
    // primary rows (integer ops)
    const unsigned jb = (WRAP && c.jb > jb_wrap) ? c.jb - (unsigned)nt : c.jb;
    return c.kb * cell_kstride + jb * cell_jstride + c.ib;
  }

  // bricked GL_QUAD cell of layer kc + dk (the r floor bits carry index - 1)
  template <bool WRAP>
  __device__ __forceinline__ unsigned quad_cell(const Cell& c, unsigned dk) const {
    const unsigned jb = (WRAP && c.jb > jb_wrap) ? c.jb - (unsigned)nt : c.jb;
    return quad_brick_index(c.kb - kMagicBits + dk, jb - kMagicBits, c.ib - kMagicBits + 1u,
                            qbrick_j, qbrick_i);
  }
  // the cell of layer kc + 1 (same row / column) from quad_cell(c, 0)
  __device__ __forceinline__ unsigned quad_cell_up(const Cell& c, unsigned idx0) const {
    return quad_next_layer(idx0, c.kb - kMagicBits, qbrick_layer);
  }
  template <bool WRAP>
  __device__ __forceinline__ unsigned oct_cell(const Cell& c) const {
    const unsigned jb = (WRAP && c.jb > jb_wrap) ? c.jb - (unsigned)nt : c.jb;
    return oct_brick_index(c.kb - kMagicBits, jb - kMagicBits, c.ib - kMagicBits + 1u,
                           brick_j, brick_i);
  }

  // the same 8 values from the plain mu layout (r/h clamp, theta modulo n_theta)
  __device__ __forceinline__ void fetch_plain(const Cell& c, float4& a, float4& b) const {
    const int i0 = (int)(c.ib - kMagicBits), g = (int)(c.jb - kMagicBits);   // r: kRMagic
    const int k0 = (int)(c.kb - kMagicBits) - 1;
    const int ia = max(i0, 0), ib1 = min(i0 + 1, nr - 1);
    const int ka = max(k0, 0), kb1 = min(k0 + 1, nh - 1);
    const int ja = (g + nt - 1) % nt, jb1 = g % nt;
    const float* p0 = mu + ((size_t)ka * nt + ja) * nr;
    const float* p1 = mu + ((size_t)ka * nt + jb1) * nr;
    const float* p2 = mu + ((size_t)kb1 * nt + ja) * nr;
    const float* p3 = mu + ((size_t)kb1 * nt + jb1) * nr;
    a = make_float4(__ldg(p0 + ia), __ldg(p0 + ib1), __ldg(p1 + ia), __ldg(p1 + ib1));
    b = make_float4(__ldg(p2 + ia), __ldg(p2 + ib1), __ldg(p3 + ia), __ldg(p3 + ib1));
  }

  __device__ __forceinline__ float sample_nearest(float x, float y, float z) const {
    const float r = sqrt_approx(fmaf(x, x, y * y));
    const float th = theta_2pi(y, x);
    const float ft1 = fmaf(th, inv_dth, 0.5f);
    const float fr = fminf(fmaxf(fmaf(r, inv_dr, -0.5f), 0.0f), nr_m1);
    const float fh = fminf(fmaxf(fmaf(z, inv_dh, h_off), 0.0f), nh_m1);
    int ir = (int)rintf(fr), ih = (int)rintf(fh), it = (int)rintf(ft1 - 1.0f);
    if (it < 0) it += nt;
    if (it >= nt) it -= nt;
    return __ldg(mu + (ih * nt + it) * nr + ir);
  }
};

struct CartGeo {
  const float* __restrict__ mu;
  const float4* __restrict__ oct;  // gather layout (ct_pack_gather_cart) or null
  bool quad;                       // oct holds GL_QUAD corner quads
  bool obrick;                     // oct holds GL_OCTB bricked 32-byte cells
  long long dbg_floats = 0;        // CT_DEBUG_BOUNDS: gather buffer length (floats)
  int nz, ny, nx;
  double vs, lo[3], hi[3];
  float inv_vs, off[3], off1[3], nx_m1, ny_m1, nz_m1;
  unsigned cell_kstride, cell_jstride;   // gather layout (nz+1, ny+1, nx+1), strides (ks, js, 1)
  double cells_layer;
  const float4* __restrict__ qraw;
  unsigned long long qtex = 0;
  unsigned brick_j, brick_i, qbrick_j, qbrick_i, qbrick_layer;

  __host__ void init(const float* m, const float* gather, const ct_cart_grid& g) {
    mu = m;
    oct = nullptr;
    nz = g.n_z; ny = g.n_y; nx = g.n_x;
    vs = g.voxel_size;
    for (int a = 0; a < 3; ++a) lo[a] = g.origin[a];
    hi[0] = g.origin[0] + g.n_x * g.voxel_size;
    hi[1] = g.origin[1] + g.n_y * g.voxel_size;
    hi[2] = g.origin[2] + g.n_z * g.voxel_size;
    inv_vs = (float)(1.0 / g.voxel_size);
    for (int a = 0; a < 3; ++a) off[a] = (float)(-g.origin[a] / g.voxel_size - 0.5);
    nx_m1 = (float)(nx - 1); ny_m1 = (float)(ny - 1); nz_m1 = (float)(nz - 1);
    for (int a = 0; a < 3; ++a) off1[a] = off[a] + 1.0f;
    const CellStrides cs = cell_strides((unsigned)ny + 1u, (unsigned)nx + 1u);
    cell_jstride = cs.js;
    cell_kstride = cs.ks;
    cells_layer = (double)(ny + 1) * (nx + 1);
    quad = gather_quad(cells_layer);
    obrick = gather_obrick(cells_layer);
    oct = gather ? cell_base(gather, quad, 0) : nullptr;
    qraw = reinterpret_cast<const float4*>(gather);
    brick_j = ((unsigned)ny + 2u) / 2u;
    brick_i = ((unsigned)nx + 2u) / 2u;
    qbrick_j = qbricks((unsigned)ny + 1u, QB_LJ);
    qbrick_i = qbricks((unsigned)nx + 1u, QB_LI);
    qbrick_layer = qbrick_j * qbrick_i * 8u;
  }

  // _kernels.py:207-231
  __device__ __forceinline__ bool interval(const double s[3], const double d[3], double& t0,
                                           double& t1) const {
    t0 = 0.0;
    t1 = 1e30;
#pragma unroll
    for (int ax = 0; ax < 3; ++ax) {
      if (fabs(d[ax]) < 1e-18) {
        if (s[ax] < lo[ax] || s[ax] > hi[ax]) return false;
      } else {
        double ta = ddiv(dsub(lo[ax], s[ax]), d[ax]);
        double tb = ddiv(dsub(hi[ax], s[ax]), d[ax]);
        if (ta > tb) { double tmp = ta; ta = tb; tb = tmp; }
        if (ta > t0) t0 = ta;
        if (tb < t1) t1 = tb;
      }
    }
    return true;
  }

  __device__ __forceinline__ bool inside(const double s[3], const double d[3], double t) const {
    double x = dadd(s[0], dmul(t, d[0]));
    double y = dadd(s[1], dmul(t, d[1]));
    double z = dadd(s[2], dmul(t, d[2]));
    return !(x < lo[0] || x > hi[0] || y < lo[1] || y > hi[1] || z < lo[2] || z > hi[2]);
  }
  // interp_cart's own outside test (_kernels.py:117-118): a counted sample can
  // still interpolate to 0 if index recovery lands outside [-.5, n-.5]
  __device__ __forceinline__ bool interp_nonzero(const double* s, const double* d,
                                                 double t) const {
    double p[3];
    for (int a = 0; a < 3; ++a) p[a] = dadd(s[a], dmul(t, d[a]));
    double f[3];
    for (int a = 0; a < 3; ++a) {
      f[a] = dsub(ddiv(dsub(p[a], lo[a]), vs), 0.5);
      double r = rint(f[a]);
      if (fabs(f[a] - r) < 1e-9) f[a] = r;
    }
    return !(f[0] < -0.5 || f[0] > nx - 0.5 || f[1] < -0.5 || f[1] > ny - 0.5 ||
             f[2] < -0.5 || f[2] > nz - 0.5);
  }

  // cell with a halo at index -1 on all three axes (see CylGeo::locate)
  __device__ __forceinline__ Cell locate(float x, float y, float z) const {
    const float fx1 = fmaf(x, inv_vs, off1[0]);
    const float fy1 = fmaf(y, inv_vs, off1[1]);
    const float fz1 = fmaf(z, inv_vs, off1[2]);
    const float tx = __fadd_rd(fx1, 8388608.0f);
    const float ty = __fadd_rd(fy1, 8388608.0f);
    const float tz = __fadd_rd(fz1, 8388608.0f);
    Cell c;
    c.w0 = fx1 - (tx - 8388608.0f);
    c.w1 = fy1 - (ty - 8388608.0f);
    c.w2 = fz1 - (tz - 8388608.0f);
    c.ib = __float_as_uint(tx);
    c.jb = __float_as_uint(ty);
    c.kb = __float_as_uint(tz);
    return c;
  }

  __device__ __forceinline__ void setup_ray(const double e[3], const double inc[3], int,
                                            RayF& ry) const {
    ry.ex = (float)e[0]; ry.ey = (float)e[1]; ry.ez = (float)e[2];
    ry.ix = (float)inc[0]; ry.iy = (float)inc[1]; ry.iz = (float)inc[2];
    ry.wrap = false;
  }
  __device__ __forceinline__ Cell locate1(float k, const RayF& ry) const {
    return locate(fmaf(k, ry.ix, ry.ex), fmaf(k, ry.iy, ry.ey), fmaf(k, ry.iz, ry.ez));
  }

  __device__ __forceinline__ void locate2(f32x2 K, const RayF& ry, Cell& ca, Cell& cb) const {
    const f32x2 X = fma2(K, dup2(ry.ix), dup2(ry.ex)), Y = fma2(K, dup2(ry.iy), dup2(ry.ey));
    const f32x2 Z = fma2(K, dup2(ry.iz), dup2(ry.ez));
    const f32x2 IV = dup2(inv_vs);
    const f32x2 FX = fma2(X, IV, dup2(off1[0])), FY = fma2(Y, IV, dup2(off1[1]));
    const f32x2 FZ = fma2(Z, IV, dup2(off1[2]));
    const f32x2 BIG = dup2(8388608.0f);
    const f32x2 TX = add2_rd(FX, BIG), TY = add2_rd(FY, BIG), TZ = add2_rd(FZ, BIG);
    upk(sub2(FX, sub2(TX, BIG)), ca.w0, cb.w0);
    upk(sub2(FY, sub2(TY, BIG)), ca.w1, cb.w1);
    upk(sub2(FZ, sub2(TZ, BIG)), ca.w2, cb.w2);
    float t0, t1;
    upk(TX, t0, t1);
    ca.ib = __float_as_uint(t0); cb.ib = __float_as_uint(t1);
    upk(TY, t0, t1);
    ca.jb = __float_as_uint(t0); cb.jb = __float_as_uint(t1);
    upk(TZ, t0, t1);
    ca.kb = __float_as_uint(t0); cb.kb = __float_as_uint(t1);
  }

  template <bool WRAP>
  __device__ __forceinline__ unsigned gather_index(const Cell& c) const {
    return c.kb * cell_kstride + c.jb * cell_jstride + c.ib;
  }
  template <bool WRAP>
  __device__ __forceinline__ unsigned quad_cell(const Cell& c, unsigned dk) const {
    return quad_brick_index(c.kb - kMagicBits + dk, c.jb - kMagicBits, c.ib - kMagicBits,
                            qbrick_j, qbrick_i);
  }
  __device__ __forceinline__ unsigned quad_cell_up(const Cell& c, unsigned idx0) const {
    return quad_next_layer(idx0, c.kb - kMagicBits, qbrick_layer);
  }
  template <bool WRAP>
  __device__ __forceinline__ unsigned oct_cell(const Cell& c) const {
    return oct_brick_index(c.kb - kMagicBits, c.jb - kMagicBits, c.ib - kMagicBits, brick_j,
                           brick_i);
  }

  __device__ __forceinline__ void fetch_plain(const Cell& c, float4& a, float4& b) const {
    const int i0 = (int)(c.ib - kMagicBits) - 1, j0 = (int)(c.jb - kMagicBits) - 1;
    const int k0 = (int)(c.kb - kMagicBits) - 1;
    const int ia = max(i0, 0), ib1 = min(i0 + 1, nx - 1);
    const int ja = max(j0, 0), jb1 = min(j0 + 1, ny - 1);
    const int ka = max(k0, 0), kb1 = min(k0 + 1, nz - 1);
    const float* p0 = mu + ((size_t)ka * ny + ja) * nx;
    const float* p1 = mu + ((size_t)ka * ny + jb1) * nx;
    const float* p2 = mu + ((size_t)kb1 * ny + ja) * nx;
    const float* p3 = mu + ((size_t)kb1 * ny + jb1) * nx;
    a = make_float4(__ldg(p0 + ia), __ldg(p0 + ib1), __ldg(p1 + ia), __ldg(p1 + ib1));
    b = make_float4(__ldg(p2 + ia), __ldg(p2 + ib1), __ldg(p3 + ia), __ldg(p3 + ib1));
  }

  __device__ __forceinline__ float sample_nearest(float x, float y, float z) const {
    const float fx = fminf(fmaxf(fmaf(x, inv_vs, off[0]), 0.0f), nx_m1);
    const float fy = fminf(fmaxf(fmaf(y, inv_vs, off[1]), 0.0f), ny_m1);
    const float fz = fminf(fmaxf(fmaf(z, inv_vs, off[2]), 0.0f), nz_m1);
    return __ldg(mu + ((int)rintf(fz) * ny + (int)rintf(fy)) * nx + (int)rintf(fx));
  }
};

int check_cyl(const ct_cyl_grid* g) {
  if (!g || g->n_h < 1 || g->n_theta < 1 || g->n_r < 1 || !(g->radius > 0) || !(g->height > 0))
    return set_err(CT_ERR_ARG, "bad cylindrical grid");
  if ((int64_t)g->n_h * g->n_theta * g->n_r >= (int64_t)1 << 31)
    return set_err(CT_ERR_ARG, "grid has >= 2^31 voxels");
  return CT_OK;
}
int check_cart(const ct_cart_grid* g) {
  if (!g || g->n_z < 1 || g->n_y < 1 || g->n_x < 1 || !(g->voxel_size > 0))
    return set_err(CT_ERR_ARG, "bad Cartesian grid");
  if ((int64_t)g->n_z * g->n_y * g->n_x >= (int64_t)1 << 31)
    return set_err(CT_ERR_ARG, "grid has >= 2^31 voxels");
  return CT_OK;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
  return x;
}
__device__ __forceinline__ double warp_max(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x = fmax(x, __shfl_xor_sync(0xffffffffu, x, o));
  return x;
}

unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace
