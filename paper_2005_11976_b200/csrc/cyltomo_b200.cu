// cyltomo_b200.cu -- sm_100a kernels + C-ABI for the cone-beam FP / BP / SART
// hot path (see include/cyltomo_b200.h for the contract, DESIGN.md for the
// data layout and rooflines).
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
#include "cyltomo_b200.h"

#include <cuda_runtime.h>
#include <limits.h>
#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

namespace {

#ifndef CT_ATAN_TERMS
#define CT_ATAN_TERMS 7          // 2 atan polynomial terms (7: 4.8e-7 rad; 8: 5.7e-8 rad)
#endif
constexpr double kPi = 3.141592653589793;
constexpr double kTwoPi = 2.0 * kPi;
constexpr float kTwoPiF = 6.28318530717958647692f;

thread_local char g_err[512] = "";

int set_err(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    snprintf(g_err, sizeof g_err, "%s: %s", what, cudaGetErrorString(e));
    return CT_ERR_CUDA;
  }
  return CT_OK;
}

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
__device__ __forceinline__ float trilinear_eval(float4 ca, float4 cb, float wr, float wt, float wh) {
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

// Large volumes use 16-byte per-layer bilinear cells (GL_QUAD) instead of the
// 32-byte trilinear cells: half the bytes per h layer, so more of the band of
// layers a wave of rays works on stays in L2, for one more load and two f32x2
// subtractions per cell entered.  Measured (A/B): C5 -23.5 %, C4-cyl equal,
// C4-cart (8.4 MB layers) +22 %, C2 (4.2 MB layers) +15 %; hence layers above
// 10 MB.  CT_GATHER_QUAD=0/1 overrides.
inline bool gather_quad(unsigned ks) {
  const char* e = getenv("CT_GATHER_QUAD");
  if (e && *e) return e[0] == '1';
  return 32.0 * ks > 10.0e6;
}

struct CylGeo {
  const float* __restrict__ mu;
  const float4* __restrict__ oct;  // gather layout (ct_pack_gather_cyl) or null
  bool quad;                       // oct holds GL_QUAD corner quads
  int nh, nt, nr;
  double radius, half_h;
  // fp32 sampling constants
  float inv_dr, inv_dth, inv_dh, h_off, h_off1, nr_m1, nh_m1;
  float tc[8];   // 2 atan polynomial coefficients times n_theta / (2 pi)
  // gather layout: cells (nh+1, nt+1, nr+1), strides (ks, js, 1)
  unsigned cell_kstride, cell_jstride, jb_wrap;

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
    cell_jstride = (unsigned)g.n_r + 1u;
    cell_kstride = gather_layer_stride((unsigned)gather_rows(g.n_theta), cell_jstride);
    quad = gather_quad(cell_kstride);
    // the r floor bits carry index - 1 (kRMagic): the base is one cell on
    oct = gather ? reinterpret_cast<const float4*>(gather) + (quad ? 1 : 2) : nullptr;
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
  __device__ __forceinline__ int gather_index(const Cell& c) const {
    // WRAP (rays crossing theta = 2 pi): rows past n_theta wrap onto the
    // primary rows (integer ops)
    const unsigned jb = (WRAP && c.jb > jb_wrap) ? c.jb - (unsigned)nt : c.jb;
    return (int)(c.kb * cell_kstride + jb * cell_jstride + c.ib);
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
  int nz, ny, nx;
  double vs, lo[3], hi[3];
  float inv_vs, off[3], off1[3], nx_m1, ny_m1, nz_m1;
  unsigned cell_kstride, cell_jstride;   // gather layout (nz+1, ny+1, nx+1), strides (ks, js, 1)

  __host__ void init(const float* m, const float* gather, const ct_cart_grid& g) {
    mu = m;
    oct = reinterpret_cast<const float4*>(gather);
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
    cell_jstride = (unsigned)nx + 1u;
    cell_kstride = gather_layer_stride((unsigned)ny + 1u, cell_jstride);
    quad = gather_quad(cell_kstride);
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
  __device__ __forceinline__ int gather_index(const Cell& c) const {
    return (int)(c.kb * cell_kstride + c.jb * cell_jstride + c.ib);
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

// ---------------------------------------------------------------------------
// forward projection
// ---------------------------------------------------------------------------
enum FpEpi { EPI_PROJECT = 0, EPI_CORR = 1, EPI_RESID = 2, EPI_ROWMAX = 3 };

// FP volume layouts: plain mu, the 32-byte polynomial cells (ct_pack_gather_*),
// or 16-byte corner quads per h layer (large volumes; see gather_quad())
enum FpLayout { GL_PLAIN = 0, GL_OCT = 1, GL_QUAD = 2 };

// block = FP_WX x FP_WY warps, each warp a pixel patch (tile_ww x tile_wh rays)
#ifndef CT_FP_WX
#define CT_FP_WX 4
#endif
#ifndef CT_FP_WY
#define CT_FP_WY 1
#endif
#ifndef CT_FP_CHAINS
#define CT_FP_CHAINS 2           // independent gather chains per ray chunk (2 or 4)
#endif
#ifndef CT_FP_UNROLL
#define CT_FP_UNROLL 2           // main march loop unroll
#endif
#ifndef CT_FP_MAXREG
#define CT_FP_MAXREG 64          // 32 warps/SM
#endif
#ifndef CT_FP_WW1
#define CT_FP_WW1 4              // warp patch width at one lane per ray
#endif
constexpr int FP_WX = CT_FP_WX, FP_WY = CT_FP_WY, FP_CHAINS = CT_FP_CHAINS, FP_UNROLL = CT_FP_UNROLL;
static_assert(FP_CHAINS == 2 || FP_CHAINS == 4, "FP_CHAINS");
constexpr int FP_THREADS = 32 * FP_WX * FP_WY;

template <class Geo>
struct FpArgs {
  Geo geo;
  const ct_ray_view* __restrict__ views;
  const int32_t* __restrict__ view_ids;
  int rows, cols, ss;
  int lanes;            // K lanes per ray (lanes_for(rows, cols))
  double step;
  const float* __restrict__ p_meas;
  const double* __restrict__ row_thr;
  float* __restrict__ out0;
  float* __restrict__ out1;
  double* __restrict__ red;  // residual partials / per-view max_row
};

// Lanes per ray.  Small detectors cannot fill 148 SMs with one thread per
// ray, so each ray's samples are split into K contiguous chunks on K adjacent
// lanes and summed with a fixed shuffle tree.  K is a function of the detector
// size only, so every FP mode (projection, correction, residual; one view or a
// batch) produces identical bits for the same ray.
__host__ __device__ inline int lanes_for(int rows, int cols) {
#ifdef CT_FORCE_LANES
  return CT_FORCE_LANES;
#endif
  const long long px = (long long)rows * cols;
  return px >= 131072 ? 1 : px >= 65536 ? 2 : px >= 32768 ? 4 : 8;
}
// warp pixel patch: K=1 8x4, K=2 4x4, K=4 4x2, K=8 2x2; block = FP_WX x FP_WY warps
__host__ __device__ inline int tile_ww(int K) { return K == 1 ? CT_FP_WW1 : (K == 8 ? 2 : 4); }
__host__ __device__ inline int tile_wh(int K) { return (32 / K) / tile_ww(K); }

// Linear-interpolation march of samples [k, k_end) of one ray (+ the last
// sample k_last when with_last), returning the fp32 sum of the values.
template <class Geo, int OCT, bool WRAP>
__device__ __forceinline__ float march_linear(const Geo& geo, const RayF& ry, int k, int k_end,
                                              bool with_last, float k_last) {
  // Linear interpolation.  OCT: consecutive samples are half a voxel apart, so
  // a sample in the same cell as its predecessor skips its (predicated-off)
  // 32-byte load and reuses the live cell.  Plain: the same 8 values from mu.
  // Same cells, weights and summation grouping either way.
  //
  // The chunk is marched as FP_CHAINS independent chains over consecutive
  // sub-ranges, each with its own live cell: the chains' gathers are in
  // flight together (a single chain serialises load -> evaluate -> next load
  // through its cell registers), and one f32x2 locate serves two chains.
  struct Chain {
    int prev = INT_MIN;   // no cell (indices are >= -1)
    float4 pa = make_float4(0.f, 0.f, 0.f, 0.f), pb = make_float4(0.f, 0.f, 0.f, 0.f);
    float sum = 0.0f;
  };
  auto value = [&](Chain& ch, const Cell& c) -> float {
    if (OCT == GL_OCT) {
      const int idx = geo.template gather_index<WRAP>(c);
      // signed: the cylindrical r bits make the first cell's index -1 (kRMagic)
      if (idx != ch.prev) ld_cell(geo.oct + 2 * (ptrdiff_t)idx, ch.pa, ch.pb);
      ch.prev = idx;   // (unconditional: equal when not reloaded; no predicated move)
      return trilinear_eval(ch.pa, ch.pb, c.w0, c.w1, c.w2);
    }
    if (OCT == GL_QUAD) {
      // bilinear layers k, k+1 of the cell; the h terms are their
      // difference (two f32x2 subtractions)
      const int idx = geo.template gather_index<WRAP>(c);
      if (idx != ch.prev) {
        const float4 a = ld_vquad(geo.oct + (ptrdiff_t)idx);
        const float4 b = ld_vquad(geo.oct + (ptrdiff_t)idx + geo.cell_kstride);
        ch.pa = a;
        float x0, x1, y0, y1;
        upk(sub2(pk(b.x, b.y), pk(a.x, a.y)), x0, x1);
        upk(sub2(pk(b.z, b.w), pk(a.z, a.w)), y0, y1);
        ch.pb = make_float4(x0, x1, y0, y1);
      }
      ch.prev = idx;
      return trilinear_eval(ch.pa, ch.pb, c.w0, c.w1, c.w2);
    }
    float4 a, b, ca, cb;
    geo.fetch_plain(c, a, b);
    trilinear_coeffs(a, b, ca, cb);
    return trilinear_eval(ca, cb, c.w0, c.w1, c.w2);
  };
  constexpr int NC = FP_CHAINS;
  Chain ch[NC];
  int kc[NC], ke[NC];
  {
    const int len = k_end - k;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      kc[c] = k + (c * len) / NC;
      ke[c] = k + ((c + 1) * len) / NC;
    }
  }
  // every chain has >= len/NC - 1 samples; 4 samples per iteration
  const int iters = ((k_end - k) / NC) / (4 / NC);
  f32x2 kf01 = pk((float)kc[0], (float)kc[1]);
#pragma unroll FP_UNROLL
  for (int it = 0; it < iters; ++it) {
    Cell c0, c1, c2, c3;
    if (NC == 2) {
      // float sample counters (exact below 2^24): no int->float conversions
      geo.locate2(kf01, ry, c0, c1);
      geo.locate2(add2(kf01, dup2(1.0f)), ry, c2, c3);
      kf01 = add2(kf01, dup2(2.0f));
      const float a0 = value(ch[0], c0);
      const float b0 = value(ch[1], c1);
      const float a1 = value(ch[0], c2);
      const float b1 = value(ch[1], c3);
      ch[0].sum += a0 + a1;
      ch[1].sum += b0 + b1;
    } else {
      geo.locate2(pk((float)kc[0], (float)kc[1]), ry, c0, c1);
      geo.locate2(pk((float)kc[NC - 2], (float)kc[NC - 1]), ry, c2, c3);
      ch[0].sum += value(ch[0], c0);
      ch[1].sum += value(ch[1], c1);
      ch[NC - 2].sum += value(ch[NC - 2], c2);
      ch[NC - 1].sum += value(ch[NC - 1], c3);
#pragma unroll
      for (int c = 0; c < NC; ++c) ++kc[c];
    }
  }
  if (NC == 2) {
    kc[0] += 2 * iters;
    kc[1] += 2 * iters;
  }
#pragma unroll
  for (int c = 0; c < NC; ++c)
    for (; kc[c] < ke[c]; ++kc[c]) ch[c].sum += value(ch[c], geo.locate1((float)kc[c], ry));
  float sum = ch[0].sum;
#pragma unroll
  for (int c = 1; c < NC; ++c) sum += ch[c].sum;
  if (with_last) sum += value(ch[NC - 1], geo.locate1(k_last, ry));
  return sum;
}

// One sub-ray, chunk `chunk` of `K`: returns this chunk's in-support sample
// count and adds the fp32 sum of its interpolated values into acc (COUNT_ONLY:
// chunk 0 returns the whole ray's count, without marching).
template <class Geo, bool NEAREST, int OCT, bool COUNT_ONLY>
__device__ __forceinline__ int march(const Geo& geo, const ct_ray_view& v, double cu, double cv,
                                     double step, float& acc, int chunk, int K) {
  double d[3];
  subray_dir(v, cu, cv, d);
  double t0, t1;
  if (!geo.interval(v.src, d, t0, t1)) return 0;
  if (t1 <= t0) return 0;
  const int n = (int)ceil(ddiv(dsub(t1, t0), step));
  const double t_last = dadd(t0, dmul((double)(n - 1) + 0.5, step));
  const bool last_in = geo.inside(v.src, d, t_last);
  if (COUNT_ONLY) return chunk == 0 ? n - 1 + (last_in ? 1 : 0) : 0;
  // fp32 march relative to the first sample position
  const double ts = dadd(t0, dmul(0.5, step));
  RayF ry;
  {
    double e[3], inc[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      e[a] = v.src[a] + ts * d[a];
      inc[a] = step * d[a];
    }
    geo.setup_ray(e, inc, n, ry);
  }
  const int n_int = n - 1;
  // interior samples [k, k_end) of this chunk; the last sample goes to chunk K-1
  int k = (chunk * n_int) / K;
  const int k_end = ((chunk + 1) * n_int) / K;
  const bool own_last = chunk == K - 1;
  float sum = 0.0f;
  if (NEAREST) {
    for (; k + 4 <= k_end; k += 4) {
      float s4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float kq = (float)(k + q);
        s4[q] = geo.sample_nearest(fmaf(kq, ry.ix, ry.ex), fmaf(kq, ry.iy, ry.ey),
                                   fmaf(kq, ry.iz, ry.ez));
      }
      sum += (s4[0] + s4[1]) + (s4[2] + s4[3]);
    }
    for (; k < k_end; ++k) {
      const float kf = (float)k;
      sum += geo.sample_nearest(fmaf(kf, ry.ix, ry.ex), fmaf(kf, ry.iy, ry.ey),
                                fmaf(kf, ry.iz, ry.ez));
    }
    if (own_last && last_in && geo.interp_nonzero(v.src, d, t_last)) {
      const float kf = (float)n_int;
      sum += geo.sample_nearest(fmaf(kf, ry.ix, ry.ex), fmaf(kf, ry.iy, ry.ey),
                                fmaf(kf, ry.iz, ry.ez));
    }
    acc += sum;
    return (k_end - (chunk * n_int) / K) + ((own_last && last_in) ? 1 : 0);
  }
  const bool with_last = own_last && last_in && geo.interp_nonzero(v.src, d, t_last);
  // rays crossing theta = 2 pi need the wrapped cell index; the choice is
  // warp-uniform so the two loop versions never diverge within a warp
  if (__any_sync(__activemask(), ry.wrap))
    sum = march_linear<Geo, OCT, true>(geo, ry, k, k_end, with_last, (float)n_int);
  else
    sum = march_linear<Geo, OCT, false>(geo, ry, k, k_end, with_last, (float)n_int);
  acc += sum;
  return (k_end - (chunk * n_int) / K) + ((own_last && last_in) ? 1 : 0);
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

template <class Geo, int EPI, bool NEAREST, int OCT>
__global__ void __maxnreg__(CT_FP_MAXREG) fp_kernel(const FpArgs<Geo> a) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int K = a.lanes;
  const int ww = tile_ww(K), wh = tile_wh(K);
  const int chunk = lane & (K - 1);
  const int rslot = lane / K;
  // each warp covers a ww x wh pixel patch, the block FP_WX x FP_WY warps
  const int col = blockIdx.x * (FP_WX * ww) + (warp % FP_WX) * ww + rslot % ww;
  const int row = blockIdx.z * (FP_WY * wh) + (warp / FP_WX) * wh + rslot / ww;
  const int b = blockIdx.y;
  const int vid = a.view_ids ? a.view_ids[b] : b;
  const bool active = row < a.rows && col < a.cols;
  const size_t npix = (size_t)a.rows * a.cols;
  const size_t pix = (size_t)row * a.cols + col;

  float acc = 0.0f;
  int count = 0;
  if (active && a.ss == 1) {
    // one sub-ray at the pixel centre ((0 + .5)/1 - .5 = 0 exactly): the view
    // basis is dead after the per-ray setup, keeping the march loop's
    // register footprint small
    count = march<Geo, NEAREST, OCT, EPI == EPI_ROWMAX>(a.geo, a.views[vid], (double)col,
                                                       (double)row, a.step, acc, chunk, K);
  } else if (active) {
    const ct_ray_view& v = a.views[vid];
    const int ss = a.ss;
    for (int sv = 0; sv < ss; ++sv) {
      const double off_v = dsub(ddiv((double)sv + 0.5, (double)ss), 0.5);
      for (int su = 0; su < ss; ++su) {
        const double off_u = dsub(ddiv((double)su + 0.5, (double)ss), 0.5);
        count += march<Geo, NEAREST, OCT, EPI == EPI_ROWMAX>(
            a.geo, v, dadd((double)col, off_u), dadd((double)row, off_v), a.step, acc, chunk, K);
      }
    }
  }
  if (K > 1) {
    // fixed-order tree over the K chunks of a ray (lanes of a ray are adjacent)
    for (int o = 1; o < K; o <<= 1) {
      acc += __shfl_xor_sync(0xffffffffu, acc, o);
      count += __shfl_xor_sync(0xffffffffu, count, o);
    }
  }
  const bool lead = chunk == 0;   // writes the ray's outputs
  const double inv_ss2 = ddiv(1.0, (double)(a.ss * a.ss));
  // out_w = wacc * step * inv_ss2, out_p = acc * step * inv_ss2 (_kernels.py:292-293)
  const double w64 = dmul(dmul((double)count, a.step), inv_ss2);
  const double p64 = (double)acc * a.step * inv_ss2;

  if (EPI == EPI_PROJECT) {
    if (active && lead) {
      a.out0[(size_t)b * npix + pix] = (float)p64;
      if (a.out1) a.out1[(size_t)b * npix + pix] = (float)w64;
    }
  } else if (EPI == EPI_CORR) {
    if (active && lead) {
      float c = 0.0f;
      if (w64 > a.row_thr[vid]) {
        const float pm = a.p_meas[(size_t)vid * npix + pix];
        c = (pm - (float)p64) / (float)w64;
      }
      a.out0[(size_t)b * npix + pix] = c;
    }
  } else {
    double x = 0.0;
    if (active && lead) {
      if (EPI == EPI_RESID) {
        // compare with the fp32 simulation, i.e. what a stored projection of
        // this volume holds: consistent data gives exactly 0, as in the reference
        const double r = (double)a.p_meas[(size_t)vid * npix + pix] - (double)(float)p64;
        x = r * r;
      } else {
        x = w64;
      }
    }
    __shared__ double sred[FP_THREADS / 32];
    x = (EPI == EPI_RESID) ? warp_sum(x) : warp_max(x);
    if (lane == 0) sred[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = sred[0];
      for (int w = 1; w < FP_THREADS / 32; ++w)
        t = (EPI == EPI_RESID) ? t + sred[w] : fmax(t, sred[w]);
      if (EPI == EPI_RESID) {
        const size_t blk = ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        a.red[blk] = t;
      } else {
        // non-negative doubles order like their bit patterns
        atomicMax(reinterpret_cast<unsigned long long*>(a.red + b),
                  (unsigned long long)__double_as_longlong(t));
      }
    }
  }
}

// Deterministic second stage: fixed-order sum of the per-block partials.
__global__ void __launch_bounds__(1024) sum_partials_kernel(const double* __restrict__ part,
                                                            int64_t n, double* accum) {
  __shared__ double s[32];
  double x = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) x += part[i];
  x = warp_sum(x);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = x;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    *accum += t;
  }
}

dim3 fp_grid(const ct_batch& b) {
  const int K = lanes_for(b.det_rows, b.det_cols);
  const int tw = FP_WX * tile_ww(K), th = FP_WY * tile_wh(K);
  return dim3((b.det_cols + tw - 1) / tw, b.n_batch, (b.det_rows + th - 1) / th);
}

int check_batch(const ct_batch* b, const void* views, const ct_sampling* s) {
  if (!b || !views || !s) return set_err(CT_ERR_ARG, "null batch/views/sampling");
  if (b->n_batch < 1 || b->n_batch > 65535 || b->det_rows < 1 || b->det_cols < 1 ||
      fp_grid(*b).z > 65535)
    return set_err(CT_ERR_ARG, "bad batch dimensions");
  if (!(s->step > 0.0) || s->supersample < 1) return set_err(CT_ERR_ARG, "bad sampling");
  return CT_OK;
}

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

template <class Geo, int EPI>
int launch_fp(const Geo& geo, const ct_ray_view* views, const ct_batch& b, const ct_sampling& s,
              const float* p_meas, const double* thr, float* o0, float* o1, double* red,
              cudaStream_t st) {
  FpArgs<Geo> a;
  a.geo = geo;
  a.views = views;
  a.view_ids = b.view_ids;
  a.rows = b.det_rows;
  a.cols = b.det_cols;
  a.ss = s.supersample;
  a.lanes = lanes_for(b.det_rows, b.det_cols);
  a.step = s.step;
  a.p_meas = p_meas;
  a.row_thr = thr;
  a.out0 = o0;
  a.out1 = o1;
  a.red = red;
  if (s.nearest)
    fp_kernel<Geo, EPI, true, GL_PLAIN><<<fp_grid(b), FP_THREADS, 0, st>>>(a);
  else if (EPI != EPI_ROWMAX && geo.oct && geo.quad)
    fp_kernel<Geo, EPI, false, GL_QUAD><<<fp_grid(b), FP_THREADS, 0, st>>>(a);
  else if (EPI != EPI_ROWMAX && geo.oct)
    fp_kernel<Geo, EPI, false, GL_OCT><<<fp_grid(b), FP_THREADS, 0, st>>>(a);
  else
    fp_kernel<Geo, EPI, false, GL_PLAIN><<<fp_grid(b), FP_THREADS, 0, st>>>(a);
  return check_launch("fp_kernel");
}

// ---------------------------------------------------------------------------
// back-projection
// ---------------------------------------------------------------------------
enum BpMode { BP_ACC = 0, BP_WRITE = 1, BP_UPDATE = 2 };

#ifndef CT_BP_THREADS
#define CT_BP_THREADS 256
#endif
constexpr int BP_THREADS = CT_BP_THREADS;
#ifndef CT_BP_UNROLL
#define CT_BP_UNROLL 4
#endif
constexpr int BP_UNROLL = CT_BP_UNROLL;
#ifndef CT_BP_MIN_BLOCKS
#define CT_BP_MIN_BLOCKS 8       // 32 registers, 64 warps/SM (A/B: 4-8)
#endif
constexpr int BP_MIN_BLOCKS = CT_BP_MIN_BLOCKS;
constexpr int BP_CHUNK = 64;   // views staged in shared memory per pass
static_assert(BP_CHUNK / 2 <= 32, "slow-pair mask is 32 bits");
constexpr float BP_EDGE_EPS = 1e-3f;  // px band around the frame edge refined in fp64

// a pair of views (batch slots 2i, 2i+1), lane-interleaved for f32x2
struct __align__(16) BpPairF {
  f32x2 cphi, sphi, sod, sdd_p;   // sdd / pitch
  f32x2 u0, v0, dfloor, coff;     // u0 + 1, v0 + 1, refine floor, tap offset (u32)
};

struct CylVox {
  int nh, nt, nr;
  double dr, dth, dh, half_h;
  double rot[9], t[3];
  const double* __restrict__ trig;  // cos[nt], sin[nt]
  __host__ void init(const ct_cyl_grid& g, const double* tr) {
    nh = g.n_h; nt = g.n_theta; nr = g.n_r;
    dr = g.radius / g.n_r;
    dth = kTwoPi / g.n_theta;
    dh = g.height / g.n_h;
    half_h = 0.5 * g.height;
    for (int i = 0; i < 9; ++i) rot[i] = g.rot[i];
    for (int i = 0; i < 3; ++i) t[i] = g.t[i];
    trig = tr;
  }
  __host__ __device__ int64_t count() const { return (int64_t)nh * nt * nr; }
  // voxel centre, object -> world (_kernels.py:396-406), reference op order
  __device__ __forceinline__ void world(int m, double w[3]) const {
    const int ir = m % nr;
    const int j = (m / nr) % nt;
    const int k = m / (nr * nt);
    const double r = dmul((double)ir + 0.5, dr);
    const double h = dsub(dmul((double)k + 0.5, dh), half_h);
    const double xo = dmul(r, trig[j]);
    const double yo = dmul(r, trig[nt + j]);
#pragma unroll
    for (int i = 0; i < 3; ++i)
      w[i] = dadd(dadd(dadd(dmul(rot[3 * i], xo), dmul(rot[3 * i + 1], yo)),
                       dmul(rot[3 * i + 2], h)), t[i]);
  }
};

struct CartVox {
  int nz, ny, nx;
  double vs, o[3];
  __host__ void init(const ct_cart_grid& g) {
    nz = g.n_z; ny = g.n_y; nx = g.n_x;
    vs = g.voxel_size;
    for (int i = 0; i < 3; ++i) o[i] = g.origin[i];
  }
  __host__ __device__ int64_t count() const { return (int64_t)nz * ny * nx; }
  // _kernels.py:431-437
  __device__ __forceinline__ void world(int m, double w[3]) const {
    const int i = m % nx;
    const int j = (m / nx) % ny;
    const int k = m / (nx * ny);
    w[0] = dadd(o[0], dmul((double)i + 0.5, vs));
    w[1] = dadd(o[1], dmul((double)j + 0.5, vs));
    w[2] = dadd(o[2], dmul((double)k + 0.5, vs));
  }
};

template <class Vox>
struct BpArgs {
  Vox vox;
  const float* __restrict__ corr;
  const float4* __restrict__ quads;   // bilinear footprints of corr (ct_pack_quads) or null
  const ct_det_view* __restrict__ dets;
  const int32_t* __restrict__ view_ids;
  int n_batch, rows, cols;
  float* num;
  float* den;
  ct_update upd;
};

// fp64 re-evaluation of one voxel-view with the reference's arithmetic
// (_kernels.py:407-417 + _bilinear_gather :350-377); only taken for
// footprints within BP_EDGE_EPS of the frame edge or near the source plane.
template <class Vox>
__device__ __noinline__ float2 bp_refine(const Vox& vox, int m, const ct_det_view& dv,
                                         const float* __restrict__ img, int rows, int cols) {
  float2 acc = make_float2(0.0f, 0.0f);   // (num, den) -- returned by value so the
                                          // caller's accumulators stay in registers
  double w[3];
  vox.world(m, w);                        // fp64 voxel centre, reference op order
  const double w0 = w[0], w1 = w[1], w2 = w[2];
  const double xi = dsub(dmul(dv.cphi, w0), dmul(dv.sphi, w1));
  const double yi = dadd(dmul(dv.sphi, w0), dmul(dv.cphi, w1));
  const double depth = dadd(dv.sod, yi);
  if (depth <= dmul(1e-6, dv.sod)) return acc;
  const double scale = ddiv(dv.sdd, dmul(depth, dv.pitch));
  const double u = dadd(dv.u0, dmul(xi, scale));
  const double v = dadd(dv.v0, dmul(w2, scale));
  const double fiu = floor(u), fiv = floor(v);
  const double fu = dsub(u, fiu), fv = dsub(v, fiv);
  if (!(fiu >= -2.0 && fiu <= (double)cols) || !(fiv >= -2.0 && fiv <= (double)rows)) return acc;
  const int iu = (int)fiu, iv = (int)fiv;
  for (int dvv = 0; dvv < 2; ++dvv) {
    const int rr = iv + dvv;
    if (rr < 0 || rr >= rows) continue;
    const double wv = dvv == 1 ? fv : dsub(1.0, fv);
    for (int duu = 0; duu < 2; ++duu) {
      const int cc = iu + duu;
      if (cc < 0 || cc >= cols) continue;
      const double wu = duu == 1 ? fu : dsub(1.0, fu);
      const double wt = dmul(wu, wv);
      acc.x += (float)wt * img[(size_t)rr * cols + cc];
      acc.y += (float)wt;
    }
  }
  return acc;
}

// One voxel-view off the interior fast path (frame edge, fp64 refine band,
// near the source plane): returns its (num, den) contribution.  u1 = u + 1,
// v1 = v + 1 in pixels; img is the view's correction image.
template <class Vox>
__device__ __forceinline__ float2 bp_view_slow(const BpArgs<Vox>& a, int m, int slot, float u1,
                                               float v1, float depth, float depth_floor,
                                               const float* __restrict__ img) {
  const float W1 = (float)a.cols + 1.0f, H1 = (float)a.rows + 1.0f;
  // signed distance (px) of the footprint to the boundary of the set where
  // den > 0, i.e. (-1, W) x (-1, H); near it, redo in fp64.
  const float edge_d = fminf(fminf(u1, W1 - u1), fminf(v1, H1 - v1));
  if (edge_d < BP_EDGE_EPS || depth <= depth_floor) {
    if (edge_d > -BP_EDGE_EPS || depth <= depth_floor) {
      const int vid = a.view_ids ? a.view_ids[slot] : slot;
      return bp_refine(a.vox, m, a.dets[vid], img, a.rows, a.cols);
    }
    return make_float2(0.0f, 0.0f);
  }
  int iu, iv;                                       // floor(u), floor(v) >= -1
  const float fu = u1 - floor_pos(u1, iu);
  const float fv = v1 - floor_pos(v1, iv);
  iu -= 1;
  iv -= 1;
  const float wu0 = 1.0f - fu, wv0 = 1.0f - fv;
  // frame edge: only in-bounds taps count (_kernels.py:365-376)
  const bool cu0 = iu >= 0, cu1 = iu + 1 < a.cols;
  const bool rv0 = iv >= 0, rv1 = iv + 1 < a.rows;
  const float* r0 = img + (iv * a.cols + iu);
  const float t00 = (rv0 && cu0) ? __ldg(r0) : 0.0f;
  const float t01 = (rv0 && cu1) ? __ldg(r0 + 1) : 0.0f;
  const float t10 = (rv1 && cu0) ? __ldg(r0 + a.cols) : 0.0f;
  const float t11 = (rv1 && cu1) ? __ldg(r0 + a.cols + 1) : 0.0f;
  float2 r;
  r.x = wv0 * fmaf(wu0, t00, fu * t01) + fv * fmaf(wu0, t10, fu * t11);
  r.y = ((cu0 ? wu0 : 0.0f) + (cu1 ? fu : 0.0f)) * ((rv0 ? wv0 : 0.0f) + (rv1 ? fv : 0.0f));
  return r;
}

// Voxel-driven BP (_kernels.py:380-417): one thread per voxel, the views of
// the batch staged in shared memory in pairs and projected two per f32x2
// instruction.  Interior footprints (all four taps on the detector, clear of
// the source plane) take the fast path: one 32-bit tap offset per view from
// the floor bit patterns, lerp-form bilinear in f32x2, den += 1 (the four
// weights sum to 1); everything else goes through bp_view_slow.  num / den
// accumulate per pair lane (even / odd batch slots) and are summed at the end.
template <class Vox, int MODE, bool QUADS>
__global__ void __launch_bounds__(BP_THREADS, BP_MIN_BLOCKS) bp_kernel(const __grid_constant__ BpArgs<Vox> a) {
  __shared__ BpPairF sv[BP_CHUNK / 2];
  const int64_t nvox = a.vox.count();
  const int m = blockIdx.x * BP_THREADS + threadIdx.x;
  const bool active = m < nvox;
  float xw = 0.0f, yw = 0.0f, zw = 0.0f;
  if (active) {
    double w64[3];
    a.vox.world(m, w64);
    xw = (float)w64[0];
    yw = (float)w64[1];
    zw = (float)w64[2];
  }
  const float W1 = (float)a.cols + 1.0f, H1 = (float)a.rows + 1.0f;
  const int npix = a.rows * a.cols;
  const f32x2 XW = dup2(xw), NYW = dup2(-yw), YW = dup2(yw), ZW = dup2(zw);
  const f32x2 BIG = dup2(8388608.0f);
  f32x2 NUM = dup2(0.0f), DEN = dup2(0.0f);
  int nfast = 0;   // interior voxel-views: den += 1 each

  for (int c0 = 0; c0 < a.n_batch; c0 += BP_CHUNK) {
    const int nc = min(BP_CHUNK, a.n_batch - c0);
    __syncthreads();
    if (threadIdx.x < nc) {
      const int slot = c0 + threadIdx.x;
      const int vid = a.view_ids ? a.view_ids[slot] : slot;
      const ct_det_view& d = a.dets[vid];
      float* f = reinterpret_cast<float*>(&sv[threadIdx.x >> 1]) + (threadIdx.x & 1);
      f[0] = (float)d.cphi;
      f[2] = (float)d.sphi;
      f[4] = (float)d.sod;
      f[6] = (float)(d.sdd / d.pitch);
      f[8] = (float)(d.u0 + 1.0);                      // u0 + 1, v0 + 1
      f[10] = (float)(d.v0 + 1.0);
      f[12] = (float)(2e-6 * d.sod);                   // refine band: 2x the reference floor
      // tap offset constant: element (iv, iu) of the slot's image from the
      // floor bit patterns ivb = B + iv + 1, iub = B + iu + 1 (mod 2^32)
      reinterpret_cast<unsigned*>(f)[14] =
          (unsigned)slot * (unsigned)npix - kMagicBits * ((unsigned)a.cols + 1u) -
          (unsigned)a.cols - 1u;
    }
    __syncthreads();
    if (!active) continue;
    const float* __restrict__ img0 = a.corr + (size_t)c0 * npix;
    const int np = nc >> 1;
    unsigned slow = 0;   // pairs of this chunk for the slow path (BP_CHUNK / 2 <= 32)
#pragma unroll BP_UNROLL
    for (int i = 0; i < np; ++i) {
      const BpPairF f = sv[i];
      const f32x2 XI = fma2(f.cphi, XW, mul2(f.sphi, NYW));
      const f32x2 YI = fma2(f.sphi, XW, mul2(f.cphi, YW));
      const f32x2 DEPTH = add2(f.sod, YI);
      float da, db;
      upk(DEPTH, da, db);
      const f32x2 R = pk(rcp_approx(da), rcp_approx(db));
      const f32x2 RC = fma2(R, fma2(sub2(dup2(0.0f), DEPTH), R, dup2(1.0f)), R);
      const f32x2 SC = mul2(f.sdd_p, RC);
      const f32x2 U1 = fma2(XI, SC, f.u0);
      const f32x2 V1 = fma2(ZW, SC, f.v0);
      const f32x2 WU = sub2(dup2(W1), U1), HV = sub2(dup2(H1), V1);
      float u1a, u1b, v1a, v1b, wua, wub, hva, hvb, dfa, dfb;
      upk(U1, u1a, u1b);
      upk(V1, v1a, v1b);
      upk(WU, wua, wub);
      upk(HV, hva, hvb);
      upk(f.dfloor, dfa, dfb);
      // edge_d > 1 <=> all four taps in bounds (then also clear of the band)
      const bool fast_a = fminf(fminf(u1a, wua), fminf(v1a, hva)) > 1.0f && da > dfa;
      const bool fast_b = fminf(fminf(u1b, wub), fminf(v1b, hvb)) > 1.0f && db > dfb;
      if (fast_a && fast_b) {
        const f32x2 TU = add2_rd(U1, BIG), TV = add2_rd(V1, BIG);
        const f32x2 FU = sub2(U1, sub2(TU, BIG)), FV = sub2(V1, sub2(TV, BIG));
        const uint2 tu = bits2(TU), tv = bits2(TV), co = bits2(f.coff);
        const unsigned oa = tv.x * (unsigned)a.cols + tu.x + co.x;
        const unsigned ob = tv.y * (unsigned)a.cols + tu.y + co.y;
        if (QUADS) {
          // one 16-byte footprint per view; lerp-form bilinear per lane
          const float4 qa = ld_quad(a.quads + oa), qb = ld_quad(a.quads + ob);
          float fua, fub, fva, fvb;
          upk(FU, fua, fub);
          upk(FV, fva, fvb);
          const float aa = fmaf(fua, qa.y - qa.x, qa.x), ba = fmaf(fua, qa.w - qa.z, qa.z);
          const float ab = fmaf(fub, qb.y - qb.x, qb.x), bb = fmaf(fub, qb.w - qb.z, qb.z);
          NUM = add2(NUM, pk(fmaf(fva, ba - aa, aa), fmaf(fvb, bb - ab, ab)));
        } else {
          const float* qa = a.corr + oa;
          const float* qb = a.corr + ob;
          const f32x2 T00 = pk(__ldg(qa), __ldg(qb));
          const f32x2 T01 = pk(__ldg(qa + 1), __ldg(qb + 1));
          const f32x2 T10 = pk(__ldg(qa + a.cols), __ldg(qb + a.cols));
          const f32x2 T11 = pk(__ldg(qa + a.cols + 1), __ldg(qb + a.cols + 1));
          const f32x2 A = fma2(FU, sub2(T01, T00), T00);
          const f32x2 B = fma2(FU, sub2(T11, T10), T10);
          NUM = add2(NUM, fma2(FV, sub2(B, A), A));
        }
        nfast += 2;
      } else {
        slow |= 1u << i;   // deferred: keeps the slow path out of the hot loop
      }
    }
    // the chunk's pairs with a frame-edge / refine-band / near-source view:
    // recompute the projection per view (the same fp32 ops as the pair path)
    while (slow) {
      const int i = __ffs(slow) - 1;
      slow &= slow - 1;
      const float* fp = reinterpret_cast<const float*>(&sv[i]);
#pragma unroll
      for (int l = 0; l < 2; ++l) {
        const float cphi = fp[0 + l], sphi = fp[2 + l], sod = fp[4 + l], sdd_p = fp[6 + l];
        const float u0 = fp[8 + l], v0 = fp[10 + l], dfl = fp[12 + l];
        const float xi = fmaf(cphi, xw, __fmul_rn(sphi, -yw));
        const float yi = fmaf(sphi, xw, __fmul_rn(cphi, yw));
        const float depth = __fadd_rn(sod, yi);
        const float r = rcp_approx(depth);
        const float sc = __fmul_rn(sdd_p, fmaf(r, fmaf(-depth, r, 1.0f), r));
        const float2 rr = bp_view_slow(a, m, c0 + 2 * i + l, fmaf(xi, sc, u0), fmaf(zw, sc, v0),
                                       depth, dfl, img0 + (size_t)(2 * i + l) * npix);
        NUM = add2(NUM, l == 0 ? pk(rr.x, 0.0f) : pk(0.0f, rr.x));
        DEN = add2(DEN, l == 0 ? pk(rr.y, 0.0f) : pk(0.0f, rr.y));
      }
    }
    if (nc & 1) {   // odd view of the chunk: scalar, into the even lane
      const int i = nc - 1;
      const float* fp = reinterpret_cast<const float*>(&sv[i >> 1]);
      const float cphi = fp[0], sphi = fp[2], sod = fp[4], sdd_p = fp[6];
      const float u0 = fp[8], v0 = fp[10], dfl = fp[12];
      const float xi = fmaf(cphi, xw, sphi * -yw);
      const float yi = fmaf(sphi, xw, cphi * yw);
      const float depth = sod + yi;
      const float r = rcp_approx(depth);
      const float scale = sdd_p * fmaf(r, fmaf(-depth, r, 1.0f), r);
      const float2 rr = bp_view_slow(a, m, c0 + i, fmaf(xi, scale, u0), fmaf(zw, scale, v0), depth,
                                     dfl, img0 + (size_t)i * npix);
      NUM = add2(NUM, pk(rr.x, 0.0f));
      DEN = add2(DEN, pk(rr.y, 0.0f));
    }
  }
  float num, den;
  {
    float n0, n1, d0, d1;
    upk(NUM, n0, n1);
    upk(DEN, d0, d1);
    num = n0 + n1;
    den = (d0 + d1) + (float)nfast;
  }
  if (!active) return;
  if (MODE == BP_ACC) {
    a.num[m] += num;
    if (a.den) a.den[m] += den;
  } else if (MODE == BP_WRITE) {
    a.num[m] = num;
    if (a.den) a.den[m] = den;
  } else {
    // cyltomo/recon.py:105-119: touched = den > 0 [& w != 0];
    // mu = max(mu + (relaxation * w) * num / den, 0)
    if (den > 0.0f) {
      float lw = a.upd.relaxation;
      if (a.upd.weights) {
        const float wm = a.upd.weights[m];
        if (wm == 0.0f) return;
        lw = lw * wm;
      }
      const float delta = (lw * num) / den;
      float mu = a.upd.mu[m] + delta;
      if (a.upd.nonneg) mu = fmaxf(mu, 0.0f);
      a.upd.mu[m] = mu;
    }
  }
}

template <class Vox, int MODE>
int launch_bp(const Vox& vox, const float* corr, const float* quads, const ct_det_view* dets,
              const ct_batch& b, float* num, float* den, const ct_update* upd, cudaStream_t st) {
  BpArgs<Vox> a;
  a.vox = vox;
  a.corr = corr;
  a.quads = reinterpret_cast<const float4*>(quads);
  a.dets = dets;
  a.view_ids = b.view_ids;
  a.n_batch = b.n_batch;
  a.rows = b.det_rows;
  a.cols = b.det_cols;
  a.num = num;
  a.den = den;
  if (upd) a.upd = *upd; else memset(&a.upd, 0, sizeof a.upd);
  const int64_t nvox = vox.count();
  const unsigned blocks = (unsigned)((nvox + BP_THREADS - 1) / BP_THREADS);
  if (quads)
    bp_kernel<Vox, MODE, true><<<blocks, BP_THREADS, 0, st>>>(a);
  else
    bp_kernel<Vox, MODE, false><<<blocks, BP_THREADS, 0, st>>>(a);
  return check_launch("bp_kernel");
}

__global__ void update_kernel(const float* __restrict__ num, const float* __restrict__ den,
                              int64_t offset, int64_t count, ct_update u) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const int64_t m = offset + i;
  const float d = den[i];
  if (!(d > 0.0f)) return;
  float lw = u.relaxation;
  if (u.weights) {
    const float wm = u.weights[m];
    if (wm == 0.0f) return;
    lw = lw * wm;
  }
  float mu = u.mu[m] + (lw * num[i]) / d;
  if (u.nonneg) mu = fmaxf(mu, 0.0f);
  u.mu[m] = mu;
}

__global__ void trig_kernel(int nt, double* trig) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nt) return;
  const double th = ((double)j + 0.5) * (kTwoPi / nt);
  trig[j] = cos(th);
  trig[nt + j] = sin(th);
}

// ---------------------------------------------------------------------------
// point sampling (fp64 index arithmetic with the reference's snap, fp32 data)
// ---------------------------------------------------------------------------
__device__ __forceinline__ double snap_idx(double f) {
  const double r = rint(f);
  return fabs(f - r) < 1e-9 ? r : f;
}

// _kernels.py:48-107
__device__ float interp_cyl64(const float* __restrict__ mu, int nh, int nt, int nr,
                              double radius, double height, double r, double th, double h,
                              bool nearest) {
  const double half_h = 0.5 * height;
  if (r > radius || h < -half_h || h > half_h) return 0.0f;
  const double dr = radius / nr, dth = kTwoPi / nt, dh = height / nh;
  double fr = fmin(fmax(snap_idx(r / dr - 0.5), 0.0), (double)nr - 1.0);
  double fh = fmin(fmax(snap_idx((h + half_h) / dh - 0.5), 0.0), (double)nh - 1.0);
  double ft = snap_idx(th / dth - 0.5);
  if (nearest) {
    const int ir = (int)rint(fr), ih = (int)rint(fh);
    long long it = (long long)rint(ft) % nt;
    if (it < 0) it += nt;
    return mu[((size_t)ih * nt + it) * nr + ir];
  }
  const int i0 = (int)floor(fr);
  const double wr = fr - i0;
  const int i1 = min(i0 + 1, nr - 1);
  const int k0 = (int)floor(fh);
  const double wh = fh - k0;
  const int k1 = min(k0 + 1, nh - 1);
  const double jf = floor(ft);
  const double wt = ft - jf;
  long long j0 = (long long)jf % nt;
  if (j0 < 0) j0 += nt;
  const long long j1 = j0 + 1 == nt ? 0 : j0 + 1;
  auto M = [&](int k, long long j, int i) { return (double)mu[((size_t)k * nt + j) * nr + i]; };
  const double c00 = M(k0, j0, i0) * (1.0 - wr) + M(k0, j0, i1) * wr;
  const double c01 = M(k0, j1, i0) * (1.0 - wr) + M(k0, j1, i1) * wr;
  const double c10 = M(k1, j0, i0) * (1.0 - wr) + M(k1, j0, i1) * wr;
  const double c11 = M(k1, j1, i0) * (1.0 - wr) + M(k1, j1, i1) * wr;
  const double c0 = c00 * (1.0 - wt) + c01 * wt;
  const double c1 = c10 * (1.0 - wt) + c11 * wt;
  return (float)(c0 * (1.0 - wh) + c1 * wh);
}

// _kernels.py:110-151
__device__ float interp_cart64(const float* __restrict__ mu, int nz, int ny, int nx, double vs,
                               const double o[3], double x, double y, double z, bool nearest) {
  double fx = snap_idx((x - o[0]) / vs - 0.5);
  double fy = snap_idx((y - o[1]) / vs - 0.5);
  double fz = snap_idx((z - o[2]) / vs - 0.5);
  if (fx < -0.5 || fx > nx - 0.5 || fy < -0.5 || fy > ny - 0.5 || fz < -0.5 || fz > nz - 0.5)
    return 0.0f;
  fx = fmin(fmax(fx, 0.0), nx - 1.0);
  fy = fmin(fmax(fy, 0.0), ny - 1.0);
  fz = fmin(fmax(fz, 0.0), nz - 1.0);
  if (nearest)
    return mu[((size_t)(int)rint(fz) * ny + (int)rint(fy)) * nx + (int)rint(fx)];
  const int i0 = (int)floor(fx), j0 = (int)floor(fy), k0 = (int)floor(fz);
  const double wx = fx - i0, wy = fy - j0, wz = fz - k0;
  const int i1 = min(i0 + 1, nx - 1), j1 = min(j0 + 1, ny - 1), k1 = min(k0 + 1, nz - 1);
  auto M = [&](int k, int j, int i) { return (double)mu[((size_t)k * ny + j) * nx + i]; };
  const double c00 = M(k0, j0, i0) * (1.0 - wx) + M(k0, j0, i1) * wx;
  const double c01 = M(k0, j1, i0) * (1.0 - wx) + M(k0, j1, i1) * wx;
  const double c10 = M(k1, j0, i0) * (1.0 - wx) + M(k1, j0, i1) * wx;
  const double c11 = M(k1, j1, i0) * (1.0 - wx) + M(k1, j1, i1) * wx;
  const double c0 = c00 * (1.0 - wy) + c01 * wy;
  const double c1 = c10 * (1.0 - wy) + c11 * wy;
  return (float)(c0 * (1.0 - wz) + c1 * wz);
}

__global__ void sample_cyl_kernel(const float* __restrict__ mu, ct_cyl_grid g,
                                  const double* __restrict__ rs, const double* __restrict__ ths,
                                  const double* __restrict__ hs, int64_t n, int nearest,
                                  float* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = interp_cyl64(mu, g.n_h, g.n_theta, g.n_r, g.radius, g.height, rs[i], ths[i], hs[i],
                        nearest != 0);
}

__global__ void sample_cart_kernel(const float* __restrict__ mu, ct_cart_grid g,
                                   const double* __restrict__ xs, const double* __restrict__ ys,
                                   const double* __restrict__ zs, int64_t n, int nearest,
                                   float* out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  out[i] = interp_cart64(mu, g.n_z, g.n_y, g.n_x, g.voxel_size, g.origin, xs[i], ys[i], zs[i],
                         nearest != 0);
}

// grid.py:310-319 -- target voxel centres (h_centers/theta_centers/r_centers)
__global__ void resample_cyl_kernel(const float* __restrict__ src_mu, ct_cyl_grid s,
                                    ct_cyl_grid d, int nearest, float* out) {
  const int64_t n = (int64_t)d.n_h * d.n_theta * d.n_r;
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  const int ir = (int)(m % d.n_r);
  const int j = (int)((m / d.n_r) % d.n_theta);
  const int k = (int)(m / ((int64_t)d.n_r * d.n_theta));
  const double r = (ir + 0.5) * (d.radius / d.n_r);
  const double th = (j + 0.5) * (kTwoPi / d.n_theta);
  const double h = (k + 0.5) * (d.height / d.n_h) - 0.5 * d.height;
  out[m] = interp_cyl64(src_mu, s.n_h, s.n_theta, s.n_r, s.radius, s.height, r, th, h,
                        nearest != 0);
}


// ---------------------------------------------------------------------------
// gather layout: cell m holds the trilinear polynomial coefficients of its
// 2x2x2 neighbourhood (r/h or x/y/z clamp, theta wrap) as two float4 = one
// 32-byte sector, so one FP sample is one 256-bit load instead of 8 scattered
// loads.
// ---------------------------------------------------------------------------
// one h-layer (blockIdx.y = kc) per grid row; cells past the layer's rows are
// the stride padding (zeroed, never read)
__global__ void pack_gather_cyl_kernel(const float* __restrict__ mu, int nh, int nt, int nr,
                                       unsigned ks, float4* __restrict__ oct) {
  // cells (kc, jc, ic), kc in [0, nh], jc in [0, nt], ic in [0, nr]: corner
  // (kc-1, jc-1, ic-1); index -1 is a halo (r/h: copy of 0; theta: row nt-1)
  const unsigned rem = blockIdx.x * blockDim.x + threadIdx.x;
  if (rem >= ks) return;
  const int kc = blockIdx.y;
  const size_t m = (size_t)kc * ks + rem;
  const unsigned js = (unsigned)nr + 1u;
  const int jc = (int)(rem / js), ic = (int)(rem % js);
  if (jc > nt) {
    oct[2 * m] = oct[2 * m + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const int i = max(ic - 1, 0), i1 = min(ic, nr - 1);
  const int k = max(kc - 1, 0), k1 = min(kc, nh - 1);
  const int j = (jc == 0) ? nt - 1 : jc - 1, j1 = (jc == nt) ? 0 : jc;
  auto M = [&](int kk, int jj, int ii) { return __ldg(mu + ((int64_t)kk * nt + jj) * nr + ii); };
  float4 ca, cb;
  trilinear_coeffs(make_float4(M(k, j, i), M(k, j, i1), M(k, j1, i), M(k, j1, i1)),
                   make_float4(M(k1, j, i), M(k1, j, i1), M(k1, j1, i), M(k1, j1, i1)), ca, cb);
  oct[2 * m] = ca;
  oct[2 * m + 1] = cb;
}

__global__ void pack_gather_cart_kernel(const float* __restrict__ mu, int nz, int ny, int nx,
                                        unsigned ks, float4* __restrict__ oct) {
  // cells (kc, jc, ic) in [0, n] per axis: corner (kc-1, jc-1, ic-1)
  const unsigned rem = blockIdx.x * blockDim.x + threadIdx.x;
  if (rem >= ks) return;
  const int kc = blockIdx.y;
  const size_t m = (size_t)kc * ks + rem;
  const unsigned js = (unsigned)nx + 1u;
  const int jc = (int)(rem / js), ic = (int)(rem % js);
  if (jc > ny) {
    oct[2 * m] = oct[2 * m + 1] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const int i = max(ic - 1, 0), i1 = min(ic, nx - 1);
  const int j = max(jc - 1, 0), j1 = min(jc, ny - 1);
  const int k = max(kc - 1, 0), k1 = min(kc, nz - 1);
  auto M = [&](int kk, int jj, int ii) { return __ldg(mu + ((int64_t)kk * ny + jj) * nx + ii); };
  float4 ca, cb;
  trilinear_coeffs(make_float4(M(k, j, i), M(k, j, i1), M(k, j1, i), M(k, j1, i1)),
                   make_float4(M(k1, j, i), M(k1, j, i1), M(k1, j1, i), M(k1, j1, i1)), ca, cb);
  oct[2 * m] = ca;
  oct[2 * m + 1] = cb;
}

// bilinear footprints of a correction stack: quad (v, u) = (c[v][u], c[v][u+1],
// c[v+1][u], c[v+1][u+1]) of the same image, 0 past the last row / column
// (never read: the BP's fast path only takes footprints inside the frame)
__global__ void pack_quads_kernel(const float* __restrict__ corr, int64_t n, int rows, int cols,
                                  float4* __restrict__ quads) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  const int u = (int)(m % cols), v = (int)((m / cols) % rows);
  const bool ru = u + 1 < cols, rv = v + 1 < rows;
  const float* p = corr + m;
  quads[m] = make_float4(__ldg(p), ru ? __ldg(p + 1) : 0.0f, rv ? __ldg(p + cols) : 0.0f,
                         (ru && rv) ? __ldg(p + cols + 1) : 0.0f);
}

// GL_QUAD: cell (kc, jc, ic), kc in [0, nz+1]: the bilinear polynomial
// (c0, cr, ct, crt) of layer kc-1 (clamped; -1 and n are halo copies) over
// rows jc-1, jc (theta wraps / y clamps) and columns ic-1, ic (clamped).  The
// trilinear cell of layers k, k+1 is (L_k, L_k+1 - L_k): the same fp32 ops as
// trilinear_coeffs, so GL_QUAD, GL_OCT and the plain path agree bit for bit.
template <bool CYL>
__global__ void pack_vquad_kernel(const float* __restrict__ mu, int nk, int nj, int ni,
                                  unsigned ks, float4* __restrict__ q) {
  const unsigned rem = blockIdx.x * blockDim.x + threadIdx.x;
  if (rem >= ks) return;
  const int kc = blockIdx.y;
  const size_t m = (size_t)kc * ks + rem;
  const unsigned js = (unsigned)ni + 1u;
  const int jc = (int)(rem / js), ic = (int)(rem % js);
  if (jc > nj) {
    q[m] = make_float4(0.f, 0.f, 0.f, 0.f);
    return;
  }
  const int k = min(max(kc - 1, 0), nk - 1);
  const int i = max(ic - 1, 0), i1 = min(ic, ni - 1);
  int j, j1;
  if (CYL) {
    j = (jc == 0) ? nj - 1 : jc - 1;
    j1 = (jc == nj) ? 0 : jc;
  } else {
    j = max(jc - 1, 0);
    j1 = min(jc, nj - 1);
  }
  const float* p0 = mu + ((int64_t)k * nj + j) * ni;
  const float* p1 = mu + ((int64_t)k * nj + j1) * ni;
  // the layer's bilinear coefficients (c0, cr, ct, crt), trilinear_coeffs' ops
  const float a0 = __ldg(p0 + i), a1 = __ldg(p0 + i1), a2 = __ldg(p1 + i), a3 = __ldg(p1 + i1);
  const float dr0 = a1 - a0, dr1 = a3 - a2;
  q[m] = make_float4(a0, dr0, a2 - a0, dr1 - dr0);
}

unsigned gather_ks_cyl(const ct_cyl_grid& g) {
  return gather_layer_stride((unsigned)CylGeo::gather_rows(g.n_theta), (unsigned)g.n_r + 1u);
}
unsigned gather_ks_cart(const ct_cart_grid& g) {
  return gather_layer_stride((unsigned)g.n_y + 1u, (unsigned)g.n_x + 1u);
}
// gather buffer length in floats: (n+1) layers x 8 floats, or GL_QUAD (n+2) x 4
int64_t gather_floats_cyl(const ct_cyl_grid& g) {
  const unsigned ks = gather_ks_cyl(g);
  return gather_quad(ks) ? 4 * (int64_t)(g.n_h + 2) * ks : 8 * (int64_t)(g.n_h + 1) * ks;
}
int64_t gather_floats_cart(const ct_cart_grid& g) {
  const unsigned ks = gather_ks_cart(g);
  return gather_quad(ks) ? 4 * (int64_t)(g.n_z + 2) * ks : 8 * (int64_t)(g.n_z + 1) * ks;
}

// Beer-Lambert p = -ln(I / I0) (cyltomo/projector.py:169-181), fp64 log of the
// fp32 inputs; flat field is a scalar or one image broadcast over the views.
// Any I <= 0 or I0 <= 0 sets *bad (the caller raises NonPositiveIntensity).
__global__ void line_integral_kernel(const float* __restrict__ in, int64_t n, int64_t npix,
                                     const float* __restrict__ flat, double flat_scalar,
                                     float* __restrict__ out, int* bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double I = in[i];
  const double I0 = flat ? (double)flat[i % npix] : flat_scalar;
  if (!(I > 0.0) || !(I0 > 0.0)) {
    atomicOr(bad, 1);
    out[i] = 0.0f;
    return;
  }
  out[i] = (float)(-log(I / I0));
}


// ---------------------------------------------------------------------------
// projection-image statistics for the pose step (cyltomo/imgproc.py): per-view
// min/max and numpy-compatible histograms (Otsu), threshold + square dilation
// masks, per-row foreground extents, strip profiles.  Integer atomics only
// (order-independent), so results are deterministic.
// ---------------------------------------------------------------------------
__device__ __forceinline__ unsigned ord_key(float f) {          // monotone float -> uint
  const unsigned u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float key_ord(unsigned k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7fffffffu) : ~k);
}

__global__ void minmax_kernel(const float* __restrict__ img, int64_t npix, unsigned* mn,
                              unsigned* mx) {
  const int v = blockIdx.y;
  const float* p = img + (int64_t)v * npix;
  unsigned lo = 0xffffffffu, hi = 0u;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    const unsigned k = ord_key(p[i]);
    lo = min(lo, k);
    hi = max(hi, k);
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(mn + v, lo);
    atomicMax(mx + v, hi);
  }
}

__global__ void key_to_float_kernel(unsigned* k, int n) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) k[i] = __float_as_uint(key_ord(k[i]));
}

// np.histogram(x, bins, range=(lo, hi)) for one view per blockIdx.y: the same
// fp64 index arithmetic and edge corrections as numpy's uniform-bin path
__global__ void histogram_kernel(const float* __restrict__ img, int64_t npix,
                                 const double* __restrict__ lo, const double* __restrict__ hi,
                                 int bins, unsigned* __restrict__ counts) {
  extern __shared__ unsigned sh[];
  const int v = blockIdx.y;
  for (int b = threadIdx.x; b < bins; b += blockDim.x) sh[b] = 0u;
  __syncthreads();
  const double a = lo[v], z = hi[v];
  const double span = __dsub_rn(z, a);
  const double stepw = __ddiv_rn(span, (double)bins);  // linspace(a, z, bins+1) spacing
  const float* p = img + (int64_t)v * npix;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < npix;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double x = (double)p[i];
    if (!(x >= a && x <= z)) continue;
    int idx = (int)__dmul_rn(__ddiv_rn(__dsub_rn(x, a), span), (double)bins);
    if (idx == bins) idx -= 1;
    // edges[i] = i * step + a (two roundings), edges[bins] = z (numpy linspace)
    const double e0 = __dadd_rn(__dmul_rn((double)idx, stepw), a);
    const double e1 = (idx + 1 == bins) ? z : __dadd_rn(__dmul_rn((double)(idx + 1), stepw), a);
    if (x < e0) idx -= 1;
    else if (x >= e1 && idx != bins - 1) idx += 1;
    atomicAdd(&sh[idx], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < bins; b += blockDim.x)
    if (sh[b]) atomicAdd(counts + (int64_t)v * bins + b, sh[b]);
}

// mask = dilate(img > level, radius) with a (2r+1)^2 square element
// (scipy binary_dilation with a full structure)
__global__ void threshold_dilate_kernel(const float* __restrict__ img, int rows, int cols,
                                        const double* __restrict__ level, int radius,
                                        unsigned char* __restrict__ mask) {
  const int v = blockIdx.z;
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int r = blockIdx.y * blockDim.y + threadIdx.y;
  if (r >= rows || c >= cols) return;
  const float* p = img + (int64_t)v * rows * cols;
  const float lv = __double2float_rd(level[v]);     // fp32 x > L  <=>  x > rd_f32(L)
  unsigned char on = 0;
  for (int dr = -radius; dr <= radius && !on; ++dr) {
    const int rr = r + dr;
    if (rr < 0 || rr >= rows) continue;
    for (int dc = -radius; dc <= radius; ++dc) {
      const int cc = c + dc;
      if (cc < 0 || cc >= cols) continue;
      if (p[(int64_t)rr * cols + cc] > lv) { on = 1; break; }
    }
  }
  mask[((int64_t)v * rows + r) * cols + c] = on;
}

// per row: leftmost / rightmost foreground column (-1 / -1 if none), the
// foreground being either a precomputed mask (FROM_IMAGE = false) or
// image > levels[v][l] for every ladder level l in one pass over the image;
// pixels in remove or inside an excluded (row0, row1, col0, col1) half-open
// rectangle are background (cyltomo/imgproc.py:66-81).  Output index
// (l * n_views + v) * rows + r.
constexpr int CT_MAX_LEVELS = 16;
template <bool FROM_IMAGE>
__global__ void __launch_bounds__(256) row_extents_kernel(
    const unsigned char* __restrict__ mask, const float* __restrict__ img,
    const double* __restrict__ levels, int n_levels, const unsigned char* __restrict__ remove,
    int rows, int cols, const int* __restrict__ rects, int n_rects, int* __restrict__ left,
    int* __restrict__ right) {
  const int v = blockIdx.y, r = blockIdx.x, nv = gridDim.y;
  const int64_t base = ((int64_t)v * rows + r) * cols;
  const int nl = FROM_IMAGE ? n_levels : 1;
  // for fp32 x and fp64 L:  x > L  <=>  x > rd_f32(L)  (NaN stays NaN -> false),
  // so the ladder compares run in fp32 with the reference's fp64 result
  float lv[CT_MAX_LEVELS];
  int lo[CT_MAX_LEVELS], hi[CT_MAX_LEVELS];
#pragma unroll
  for (int l = 0; l < CT_MAX_LEVELS; ++l) {
    lv[l] = (FROM_IMAGE && l < nl) ? __double2float_rd(levels[(int64_t)v * n_levels + l]) : 0.f;
    lo[l] = INT_MAX;
    hi[l] = -1;
  }
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    bool keep = !(remove && remove[base + c]);
    for (int q = 0; q < n_rects && keep; ++q)
      if (r >= rects[4 * q] && r < rects[4 * q + 1] && c >= rects[4 * q + 2] &&
          c < rects[4 * q + 3])
        keep = false;
    if (!keep) continue;
    if (FROM_IMAGE) {
      const float x = img[base + c];
#pragma unroll
      for (int l = 0; l < CT_MAX_LEVELS; ++l)
        if (l < nl && x > lv[l]) {
          lo[l] = min(lo[l], c);
          hi[l] = max(hi[l], c);
        }
    } else if (mask[base + c]) {
      lo[0] = min(lo[0], c);
      hi[0] = max(hi[0], c);
    }
  }
  __shared__ int slo[CT_MAX_LEVELS][8], shi[CT_MAX_LEVELS][8];
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
  for (int l = 0; l < CT_MAX_LEVELS; ++l) {
    if (l >= nl) break;
    int a = lo[l], b = hi[l];
    for (int o = 16; o > 0; o >>= 1) {
      a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
      b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if ((threadIdx.x & 31) == 0) { slo[l][warp] = a; shi[l][warp] = b; }
  }
  __syncthreads();
  if (threadIdx.x < nl) {
    const int l = threadIdx.x;
    int a = INT_MAX, b = -1;
    for (int w = 0; w < nw; ++w) { a = min(a, slo[l][w]); b = max(b, shi[l][w]); }
    const int64_t o = ((int64_t)l * nv + v) * rows + r;
    left[o] = (a == INT_MAX) ? -1 : a;
    right[o] = b;
  }
}

// axis endpoints from per-row extents (cyltomo/imgproc.py:97-131), one block per
// (level, view) table: first/last foreground rows, then the band corners --
// extreme columns within the band rows, ties on an extreme column resolved to
// the outermost row.  Integer work plus exact halves, so the fp64 outputs equal
// the host rule bit for bit.  out[t] = (top_u, top_v, bottom_u, bottom_v),
// status[t] = 0 ok, 1 empty, 2 fewer than two rows.
__device__ void band_corners(const int* __restrict__ L, const int* __restrict__ R, int lo, int hi,
                             int outward, double* u, double* v) {
  int cl = INT_MAX, cr = -1;
  for (int r = lo; r <= hi; ++r)
    if (L[r] >= 0) { cl = min(cl, L[r]); cr = max(cr, R[r]); }
  int vl = -1, vr = -1;
  for (int r = lo; r <= hi; ++r) {
    if (L[r] < 0) continue;
    if (L[r] == cl && (vl < 0 || outward > 0)) vl = r;   // first (top) or last (bottom)
    if (R[r] == cr && (vr < 0 || outward > 0)) vr = r;
  }
  *u = 0.5 * (double)(cl + cr);
  *v = (double)lo + 0.5 * (double)((vl - lo) + (vr - lo));
}

__global__ void axis_endpoints_kernel(const int* __restrict__ left, const int* __restrict__ right,
                                      int rows, int band, double* __restrict__ out,
                                      int* __restrict__ status) {
  const int t = blockIdx.x;
  const int* L = left + (int64_t)t * rows;
  const int* R = right + (int64_t)t * rows;
  int rmin = INT_MAX, rmax = -1;
  for (int r = threadIdx.x; r < rows; r += blockDim.x)
    if (L[r] >= 0) { rmin = min(rmin, r); rmax = max(rmax, r); }
  for (int o = 16; o > 0; o >>= 1) {
    rmin = min(rmin, __shfl_xor_sync(0xffffffffu, rmin, o));
    rmax = max(rmax, __shfl_xor_sync(0xffffffffu, rmax, o));
  }
  __shared__ int smin[32], smax[32];
  if ((threadIdx.x & 31) == 0) { smin[threadIdx.x >> 5] = rmin; smax[threadIdx.x >> 5] = rmax; }
  __syncthreads();
  if (threadIdx.x != 0) return;
  for (int w = 1; w < (int)(blockDim.x >> 5); ++w) { rmin = min(rmin, smin[w]); rmax = max(rmax, smax[w]); }
  double* o = out + 4 * (int64_t)t;
  if (rmax < 0 || rmax - rmin < 1) {
    status[t] = rmax < 0 ? 1 : 2;
    o[0] = o[1] = o[2] = o[3] = 0.0;
    return;
  }
  double tu, tv, bu, bv;
  band_corners(L, R, rmin, min(rmin + band, rmax), -1, &tu, &tv);
  band_corners(L, R, max(rmax - band, rmin), rmax, +1, &bu, &bv);
  if (tv > bv) { double a = tu; tu = bu; bu = a; a = tv; tv = bv; bv = a; }
  o[0] = tu; o[1] = tv; o[2] = bu; o[3] = bv;
  status[t] = 0;
}

// mean bilinear grey value of a strip parallel to the projected axis
// (cyltomo/imgproc.py:133-180 strip_profile); one block per view, fixed-order
// fp64 reduction.  geom[v] = (u0, v0, u1, v1, |p1 - p0|); out[v] = NaN if no
// valid sample.
__global__ void strip_profile_kernel(const float* __restrict__ img, int rows, int cols,
                                     const double* __restrict__ geom, double offset,
                                     double width, double* __restrict__ out) {
  const int v = blockIdx.x;
  const double* g = geom + 5 * v;
  const double du = __dsub_rn(g[2], g[0]), dv = __dsub_rn(g[3], g[1]);
  const double length = g[4];                      // host np.linalg.norm (exact match)
  __shared__ double ssum[32], scnt[32];
  double sum = 0.0, cnt = 0.0;
  if (length > 0.0) {
    const double ah0 = __ddiv_rn(du, length), ah1 = __ddiv_rn(dv, length);
    const double nh0 = ah1, nh1 = -ah0;
    const int nt = max(2, (int)rint(length) + 1);   // Python round(): half-even == rint
    const int nl = max(1, (int)rint(width));
    const double tstep = __ddiv_rn(length, (double)(nt - 1));
    const float* p = img + (int64_t)v * rows * cols;
    // the reference's numpy expression order, no FMA contraction
    for (int s = threadIdx.x; s < nt * nl; s += blockDim.x) {
      const int it = s / nl, il = s % nl;
      const double t = (it == nt - 1) ? length : __dmul_rn((double)it, tstep);
      const double off = __dadd_rn(offset, __dsub_rn((double)il, (nl - 1) / 2.0));
      const double u = __dadd_rn(__dadd_rn(g[0], __dmul_rn(t, ah0)), __dmul_rn(off, nh0));
      const double w = __dadd_rn(__dadd_rn(g[1], __dmul_rn(t, ah1)), __dmul_rn(off, nh1));
      if (!(u >= 0 && u <= cols - 1 && w >= 0 && w <= rows - 1)) continue;
      const int iu = cols > 1 ? min((int)u, cols - 2) : 0;
      const int iv = rows > 1 ? min((int)w, rows - 2) : 0;
      const double fu = __dsub_rn(u, (double)iu), fv = __dsub_rn(w, (double)iv);
      const double gu = __dsub_rn(1.0, fu), gv = __dsub_rn(1.0, fv);
      const int i1 = min(iu + 1, cols - 1), j1 = min(iv + 1, rows - 1);
      double val = __dmul_rn(__dmul_rn((double)p[(int64_t)iv * cols + iu], gu), gv);
      val = __dadd_rn(val, __dmul_rn(__dmul_rn((double)p[(int64_t)iv * cols + i1], fu), gv));
      val = __dadd_rn(val, __dmul_rn(__dmul_rn((double)p[(int64_t)j1 * cols + iu], gu), fv));
      val = __dadd_rn(val, __dmul_rn(__dmul_rn((double)p[(int64_t)j1 * cols + i1], fu), fv));
      sum += val;
      cnt += 1.0;
    }
  }
  sum = warp_sum(sum);
  cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0) { ssum[threadIdx.x >> 5] = sum; scnt[threadIdx.x >> 5] = cnt; }
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0, c = 0.0;
    for (int w2 = 0; w2 < (int)(blockDim.x >> 5); ++w2) { a += ssum[w2]; c += scnt[w2]; }
    out[v] = c > 0.0 ? a / c : nan("");
  }
}

unsigned blocks_for(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

int ct_abi_version(void) { return CT_ABI_VERSION; }
const char* ct_last_error(void) { return g_err; }
const char* ct_arch(void) { return "sm_100a"; }

#define CT_STREAM(s) (static_cast<cudaStream_t>(s))

int ct_fp_cyl(const float* mu, const float* gather, const ct_cyl_grid* grid, const ct_ray_view* views,
              const ct_batch* batch, const ct_sampling* s, float* out_p, float* out_w,
              ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cyl(grid))) return rc;
  if (!mu || !out_p) return set_err(CT_ERR_ARG, "null mu/out_p");
  CylGeo geo;
  geo.init(mu, gather, *grid);
  return launch_fp<CylGeo, EPI_PROJECT>(geo, views, *batch, *s, nullptr, nullptr, out_p, out_w,
                                        nullptr, CT_STREAM(stream));
}

int ct_fp_cart(const float* mu, const float* gather, const ct_cart_grid* grid, const ct_ray_view* views,
               const ct_batch* batch, const ct_sampling* s, float* out_p, float* out_w,
               ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cart(grid))) return rc;
  if (!mu || !out_p) return set_err(CT_ERR_ARG, "null mu/out_p");
  CartGeo geo;
  geo.init(mu, gather, *grid);
  return launch_fp<CartGeo, EPI_PROJECT>(geo, views, *batch, *s, nullptr, nullptr, out_p, out_w,
                                         nullptr, CT_STREAM(stream));
}

int ct_fp_cyl_correction(const float* mu, const float* gather, const ct_cyl_grid* grid, const ct_ray_view* views,
                         const ct_batch* batch, const ct_sampling* s, const float* p_meas,
                         const double* row_thr, float* corr, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cyl(grid))) return rc;
  if (!mu || !p_meas || !row_thr || !corr) return set_err(CT_ERR_ARG, "null pointer");
  CylGeo geo;
  geo.init(mu, gather, *grid);
  return launch_fp<CylGeo, EPI_CORR>(geo, views, *batch, *s, p_meas, row_thr, corr, nullptr,
                                     nullptr, CT_STREAM(stream));
}

int ct_fp_cart_correction(const float* mu, const float* gather, const ct_cart_grid* grid, const ct_ray_view* views,
                          const ct_batch* batch, const ct_sampling* s, const float* p_meas,
                          const double* row_thr, float* corr, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cart(grid))) return rc;
  if (!mu || !p_meas || !row_thr || !corr) return set_err(CT_ERR_ARG, "null pointer");
  CartGeo geo;
  geo.init(mu, gather, *grid);
  return launch_fp<CartGeo, EPI_CORR>(geo, views, *batch, *s, p_meas, row_thr, corr, nullptr,
                                      nullptr, CT_STREAM(stream));
}

int64_t ct_residual_scratch_len(const ct_batch* batch) {
  if (!batch) return 0;
  dim3 g = fp_grid(*batch);
  return (int64_t)g.x * g.y * g.z;
}

static int finish_residual(const ct_batch* batch, double* scratch, double* accum,
                           cudaStream_t st) {
  sum_partials_kernel<<<1, 1024, 0, st>>>(scratch, ct_residual_scratch_len(batch), accum);
  return check_launch("sum_partials_kernel");
}

int ct_fp_cyl_residual(const float* mu, const float* gather, const ct_cyl_grid* grid, const ct_ray_view* views,
                       const ct_batch* batch, const ct_sampling* s, const float* p_meas,
                       double* scratch, double* accum, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cyl(grid))) return rc;
  if (!mu || !p_meas || !scratch || !accum) return set_err(CT_ERR_ARG, "null pointer");
  CylGeo geo;
  geo.init(mu, gather, *grid);
  rc = launch_fp<CylGeo, EPI_RESID>(geo, views, *batch, *s, p_meas, nullptr, nullptr, nullptr,
                                    scratch, CT_STREAM(stream));
  return rc ? rc : finish_residual(batch, scratch, accum, CT_STREAM(stream));
}

int ct_fp_cart_residual(const float* mu, const float* gather, const ct_cart_grid* grid, const ct_ray_view* views,
                        const ct_batch* batch, const ct_sampling* s, const float* p_meas,
                        double* scratch, double* accum, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cart(grid))) return rc;
  if (!mu || !p_meas || !scratch || !accum) return set_err(CT_ERR_ARG, "null pointer");
  CartGeo geo;
  geo.init(mu, gather, *grid);
  rc = launch_fp<CartGeo, EPI_RESID>(geo, views, *batch, *s, p_meas, nullptr, nullptr, nullptr,
                                     scratch, CT_STREAM(stream));
  return rc ? rc : finish_residual(batch, scratch, accum, CT_STREAM(stream));
}

int ct_rowsum_max_cyl(const ct_cyl_grid* grid, const ct_ray_view* views, const ct_batch* batch,
                      const ct_sampling* s, double* max_row, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cyl(grid))) return rc;
  if (!max_row) return set_err(CT_ERR_ARG, "null max_row");
  if (cudaMemsetAsync(max_row, 0, sizeof(double) * batch->n_batch, CT_STREAM(stream)))
    return check_launch("memset");
  CylGeo geo;
  geo.init(nullptr, nullptr, *grid);
  return launch_fp<CylGeo, EPI_ROWMAX>(geo, views, *batch, *s, nullptr, nullptr, nullptr,
                                       nullptr, max_row, CT_STREAM(stream));
}

int ct_rowsum_max_cart(const ct_cart_grid* grid, const ct_ray_view* views,
                       const ct_batch* batch, const ct_sampling* s, double* max_row,
                       ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cart(grid))) return rc;
  if (!max_row) return set_err(CT_ERR_ARG, "null max_row");
  if (cudaMemsetAsync(max_row, 0, sizeof(double) * batch->n_batch, CT_STREAM(stream)))
    return check_launch("memset");
  CartGeo geo;
  geo.init(nullptr, nullptr, *grid);
  return launch_fp<CartGeo, EPI_ROWMAX>(geo, views, *batch, *s, nullptr, nullptr, nullptr,
                                        nullptr, max_row, CT_STREAM(stream));
}

static int check_bp(const float* corr, const ct_det_view* dets, const ct_batch* b) {
  if (!corr || !dets || !b) return set_err(CT_ERR_ARG, "null corr/dets/batch");
  if (b->n_batch < 1 || b->det_rows < 1 || b->det_cols < 1)
    return set_err(CT_ERR_ARG, "bad batch dimensions");
  // the BP addresses the correction stack with 32-bit element offsets
  if ((int64_t)b->n_batch * b->det_rows * b->det_cols > (int64_t)0xFFFFFFFFu)
    return set_err(CT_ERR_ARG, "BP batch too large (n_batch*rows*cols must be < 2^32)");
  return CT_OK;
}

int ct_bp_cyl(const float* corr, const float* quads, const ct_det_view* dets, const ct_batch* batch,
              const ct_cyl_grid* grid, const double* trig, float* num, float* den,
              int accumulate, ct_stream_t stream) {
  int rc = check_bp(corr, dets, batch);
  if (rc || (rc = check_cyl(grid))) return rc;
  if (!trig || !num) return set_err(CT_ERR_ARG, "null trig/num");
  CylVox vox;
  vox.init(*grid, trig);
  if (accumulate)
    return launch_bp<CylVox, BP_ACC>(vox, corr, quads, dets, *batch, num, den, nullptr, CT_STREAM(stream));
  return launch_bp<CylVox, BP_WRITE>(vox, corr, quads, dets, *batch, num, den, nullptr, CT_STREAM(stream));
}

int ct_bp_cart(const float* corr, const float* quads, const ct_det_view* dets, const ct_batch* batch,
               const ct_cart_grid* grid, float* num, float* den, int accumulate,
               ct_stream_t stream) {
  int rc = check_bp(corr, dets, batch);
  if (rc || (rc = check_cart(grid))) return rc;
  if (!num) return set_err(CT_ERR_ARG, "null num");
  CartVox vox;
  vox.init(*grid);
  if (accumulate)
    return launch_bp<CartVox, BP_ACC>(vox, corr, quads, dets, *batch, num, den, nullptr, CT_STREAM(stream));
  return launch_bp<CartVox, BP_WRITE>(vox, corr, quads, dets, *batch, num, den, nullptr, CT_STREAM(stream));
}

int ct_bp_cyl_update(const float* corr, const float* quads, const ct_det_view* dets, const ct_batch* batch,
                     const ct_cyl_grid* grid, const double* trig, const ct_update* upd,
                     ct_stream_t stream) {
  int rc = check_bp(corr, dets, batch);
  if (rc || (rc = check_cyl(grid))) return rc;
  if (!trig || !upd || !upd->mu) return set_err(CT_ERR_ARG, "null trig/update/mu");
  CylVox vox;
  vox.init(*grid, trig);
  return launch_bp<CylVox, BP_UPDATE>(vox, corr, quads, dets, *batch, nullptr, nullptr, upd,
                                      CT_STREAM(stream));
}

int ct_bp_cart_update(const float* corr, const float* quads, const ct_det_view* dets, const ct_batch* batch,
                      const ct_cart_grid* grid, const ct_update* upd, ct_stream_t stream) {
  int rc = check_bp(corr, dets, batch);
  if (rc || (rc = check_cart(grid))) return rc;
  if (!upd || !upd->mu) return set_err(CT_ERR_ARG, "null update/mu");
  CartVox vox;
  vox.init(*grid);
  return launch_bp<CartVox, BP_UPDATE>(vox, corr, quads, dets, *batch, nullptr, nullptr, upd,
                                       CT_STREAM(stream));
}

int ct_cyl_trig(const ct_cyl_grid* grid, double* trig, ct_stream_t stream) {
  int rc = check_cyl(grid);
  if (rc) return rc;
  if (!trig) return set_err(CT_ERR_ARG, "null trig");
  trig_kernel<<<blocks_for(grid->n_theta, 256), 256, 0, CT_STREAM(stream)>>>(grid->n_theta, trig);
  return check_launch("trig_kernel");
}

int ct_sart_update(const float* num, const float* den, int64_t offset, int64_t count,
                   const ct_update* upd, ct_stream_t stream) {
  if (!num || !den || !upd || !upd->mu || offset < 0 || count < 0)
    return set_err(CT_ERR_ARG, "bad update arguments");
  if (count == 0) return CT_OK;
  update_kernel<<<blocks_for(count, 256), 256, 0, CT_STREAM(stream)>>>(num, den, offset, count,
                                                                       *upd);
  return check_launch("update_kernel");
}

int ct_sample_cyl(const float* mu, const ct_cyl_grid* grid, const double* rs, const double* ths,
                  const double* hs, int64_t n, int nearest, float* out, ct_stream_t stream) {
  int rc = check_cyl(grid);
  if (rc) return rc;
  if (!mu || !rs || !ths || !hs || !out || n < 0) return set_err(CT_ERR_ARG, "bad sample args");
  if (n == 0) return CT_OK;
  sample_cyl_kernel<<<blocks_for(n, 256), 256, 0, CT_STREAM(stream)>>>(mu, *grid, rs, ths, hs, n,
                                                                       nearest, out);
  return check_launch("sample_cyl_kernel");
}

int ct_sample_cart(const float* mu, const ct_cart_grid* grid, const double* xs, const double* ys,
                   const double* zs, int64_t n, int nearest, float* out, ct_stream_t stream) {
  int rc = check_cart(grid);
  if (rc) return rc;
  if (!mu || !xs || !ys || !zs || !out || n < 0) return set_err(CT_ERR_ARG, "bad sample args");
  if (n == 0) return CT_OK;
  sample_cart_kernel<<<blocks_for(n, 256), 256, 0, CT_STREAM(stream)>>>(mu, *grid, xs, ys, zs, n,
                                                                        nearest, out);
  return check_launch("sample_cart_kernel");
}

int ct_resample_cyl_to_cyl(const float* src_mu, const ct_cyl_grid* src, const ct_cyl_grid* dst,
                           int nearest, float* dst_mu, ct_stream_t stream) {
  int rc = check_cyl(src);
  if (rc || (rc = check_cyl(dst))) return rc;
  if (!src_mu || !dst_mu) return set_err(CT_ERR_ARG, "null volume");
  const int64_t n = (int64_t)dst->n_h * dst->n_theta * dst->n_r;
  resample_cyl_kernel<<<blocks_for(n, 256), 256, 0, CT_STREAM(stream)>>>(src_mu, *src, *dst,
                                                                         nearest, dst_mu);
  return check_launch("resample_cyl_kernel");
}

int ct_line_integrals(const float* intensity, int64_t n, int64_t npix, const float* flat,
                      double flat_scalar, float* out, int* bad, ct_stream_t stream) {
  if (!intensity || !out || !bad || n < 0 || npix < 1)
    return set_err(CT_ERR_ARG, "bad line-integral arguments");
  if (n == 0) return CT_OK;
  line_integral_kernel<<<blocks_for(n, 256), 256, 0, CT_STREAM(stream)>>>(
      intensity, n, npix, flat, flat_scalar, out, bad);
  return check_launch("line_integral_kernel");
}

int64_t ct_gather_floats_cyl(const ct_cyl_grid* grid) {
  return check_cyl(grid) ? 0 : gather_floats_cyl(*grid);
}
int64_t ct_gather_floats_cart(const ct_cart_grid* grid) {
  return check_cart(grid) ? 0 : gather_floats_cart(*grid);
}

int ct_pack_gather_cyl(const float* mu, const ct_cyl_grid* grid, float* gather,
                       ct_stream_t stream) {
  int rc = check_cyl(grid);
  if (rc) return rc;
  if (!mu || !gather) return set_err(CT_ERR_ARG, "null mu/gather");
  if (reinterpret_cast<uintptr_t>(gather) % 16) return set_err(CT_ERR_ARG, "gather not 16B-aligned");
  if (grid->n_h + 2 > 65535) return set_err(CT_ERR_ARG, "gather layout: n_h + 2 > 65535");
  const unsigned ks = gather_ks_cyl(*grid);
  if (gather_quad(ks)) {
    pack_vquad_kernel<true><<<dim3(blocks_for(ks, 256), grid->n_h + 2), 256, 0, CT_STREAM(stream)>>>(
        mu, grid->n_h, grid->n_theta, grid->n_r, ks, reinterpret_cast<float4*>(gather));
    return check_launch("pack_vquad_kernel");
  }
  pack_gather_cyl_kernel<<<dim3(blocks_for(ks, 256), grid->n_h + 1), 256, 0, CT_STREAM(stream)>>>(
      mu, grid->n_h, grid->n_theta, grid->n_r, ks, reinterpret_cast<float4*>(gather));
  return check_launch("pack_gather_cyl_kernel");
}

int ct_pack_gather_cart(const float* mu, const ct_cart_grid* grid, float* gather,
                        ct_stream_t stream) {
  int rc = check_cart(grid);
  if (rc) return rc;
  if (!mu || !gather) return set_err(CT_ERR_ARG, "null mu/gather");
  if (reinterpret_cast<uintptr_t>(gather) % 16) return set_err(CT_ERR_ARG, "gather not 16B-aligned");
  if (grid->n_z + 2 > 65535) return set_err(CT_ERR_ARG, "gather layout: n_z + 2 > 65535");
  const unsigned ks = gather_ks_cart(*grid);
  if (gather_quad(ks)) {
    pack_vquad_kernel<false><<<dim3(blocks_for(ks, 256), grid->n_z + 2), 256, 0, CT_STREAM(stream)>>>(
        mu, grid->n_z, grid->n_y, grid->n_x, ks, reinterpret_cast<float4*>(gather));
    return check_launch("pack_vquad_kernel");
  }
  pack_gather_cart_kernel<<<dim3(blocks_for(ks, 256), grid->n_z + 1), 256, 0, CT_STREAM(stream)>>>(
      mu, grid->n_z, grid->n_y, grid->n_x, ks, reinterpret_cast<float4*>(gather));
  return check_launch("pack_gather_cart_kernel");
}

int64_t ct_quads_floats(const ct_batch* batch) {
  if (!batch || batch->n_batch < 1 || batch->det_rows < 1 || batch->det_cols < 1) return 0;
  return 4 * (int64_t)batch->n_batch * batch->det_rows * batch->det_cols;
}

int ct_pack_quads(const float* corr, const ct_batch* batch, float* quads, ct_stream_t stream) {
  if (!corr || !quads || !batch) return set_err(CT_ERR_ARG, "null corr/quads/batch");
  if (batch->n_batch < 1 || batch->det_rows < 1 || batch->det_cols < 1)
    return set_err(CT_ERR_ARG, "bad batch dimensions");
  const int64_t n = (int64_t)batch->n_batch * batch->det_rows * batch->det_cols;
  pack_quads_kernel<<<blocks_for(n, 256), 256, 0, CT_STREAM(stream)>>>(
      corr, n, batch->det_rows, batch->det_cols, reinterpret_cast<float4*>(quads));
  return check_launch("pack_quads_kernel");
}

// ---- projection-image statistics for the pose step --------------------------
int ct_image_minmax(const float* images, int n_views, int64_t npix, float* mn, float* mx,
                    ct_stream_t stream) {
  if (!images || !mn || !mx || n_views < 1 || npix < 1)
    return set_err(CT_ERR_ARG, "bad minmax arguments");
  cudaStream_t st = CT_STREAM(stream);
  unsigned* kmn = reinterpret_cast<unsigned*>(mn);
  unsigned* kmx = reinterpret_cast<unsigned*>(mx);
  if (cudaMemsetAsync(kmn, 0xff, sizeof(unsigned) * n_views, st) ||
      cudaMemsetAsync(kmx, 0, sizeof(unsigned) * n_views, st))
    return check_launch("memset");
  const int64_t nb = (npix + 255) / 256;
  const unsigned gx = (unsigned)(nb < 256 ? nb : 256);
  minmax_kernel<<<dim3(gx, n_views), 256, 0, st>>>(images, npix, kmn, kmx);
  key_to_float_kernel<<<blocks_for(n_views, 128), 128, 0, st>>>(kmn, n_views);
  key_to_float_kernel<<<blocks_for(n_views, 128), 128, 0, st>>>(kmx, n_views);
  return check_launch("minmax_kernel");
}

int ct_image_histogram(const float* images, int n_views, int64_t npix, const double* lo,
                       const double* hi, int bins, unsigned* counts, ct_stream_t stream) {
  if (!images || !lo || !hi || !counts || n_views < 1 || npix < 1 || bins < 1 || bins > 8192)
    return set_err(CT_ERR_ARG, "bad histogram arguments");
  cudaStream_t st = CT_STREAM(stream);
  if (cudaMemsetAsync(counts, 0, sizeof(unsigned) * (size_t)bins * n_views, st))
    return check_launch("memset");
  const int64_t nb = (npix + 255) / 256;
  const unsigned gx = (unsigned)(nb < 128 ? nb : 128);
  histogram_kernel<<<dim3(gx, n_views), 256, sizeof(unsigned) * bins, st>>>(images, npix, lo, hi,
                                                                            bins, counts);
  return check_launch("histogram_kernel");
}

int ct_threshold_dilate(const float* images, int n_views, int rows, int cols,
                        const double* levels, int radius, unsigned char* mask,
                        ct_stream_t stream) {
  if (!images || !levels || !mask || n_views < 1 || rows < 1 || cols < 1 || radius < 0 ||
      n_views > 65535)
    return set_err(CT_ERR_ARG, "bad threshold/dilate arguments");
  dim3 blk(32, 8);
  dim3 grd((cols + 31) / 32, (rows + 7) / 8, n_views);
  threshold_dilate_kernel<<<grd, blk, 0, CT_STREAM(stream)>>>(images, rows, cols, levels, radius,
                                                              mask);
  return check_launch("threshold_dilate_kernel");
}

int ct_row_extents(const unsigned char* mask, const unsigned char* remove, int n_views, int rows,
                   int cols, const int* rects, int n_rects, int* left, int* right,
                   ct_stream_t stream) {
  if (!mask || !left || !right || n_views < 1 || rows < 1 || cols < 1 || n_rects < 0 ||
      (n_rects > 0 && !rects) || n_views > 65535)
    return set_err(CT_ERR_ARG, "bad row-extent arguments");
  row_extents_kernel<false><<<dim3(rows, n_views), 256, 0, CT_STREAM(stream)>>>(
      mask, nullptr, nullptr, 1, remove, rows, cols, rects, n_rects, left, right);
  return check_launch("row_extents_kernel");
}

int ct_row_extents_levels(const float* images, const double* levels, int n_levels,
                          const unsigned char* remove, int n_views, int rows, int cols,
                          const int* rects, int n_rects, int* left, int* right,
                          ct_stream_t stream) {
  if (!images || !levels || !left || !right || n_views < 1 || rows < 1 || cols < 1 ||
      n_levels < 1 || n_levels > CT_MAX_LEVELS || n_rects < 0 || (n_rects > 0 && !rects) ||
      n_views > 65535)
    return set_err(CT_ERR_ARG, "bad row-extent arguments");
  row_extents_kernel<true><<<dim3(rows, n_views), 256, 0, CT_STREAM(stream)>>>(
      nullptr, images, levels, n_levels, remove, rows, cols, rects, n_rects, left, right);
  return check_launch("row_extents_kernel");
}

int ct_axis_endpoints(const int* left, const int* right, int n_tables, int rows, int band,
                      double* out, int* status, ct_stream_t stream) {
  if (!left || !right || !out || !status || n_tables < 1 || rows < 1 || band < 0)
    return set_err(CT_ERR_ARG, "bad axis-endpoint arguments");
  axis_endpoints_kernel<<<n_tables, 256, 0, CT_STREAM(stream)>>>(left, right, rows, band, out,
                                                                status);
  return check_launch("axis_endpoints_kernel");
}

int ct_strip_profiles(const float* images, int n_views, int rows, int cols, const double* axes,
                      double offset, double width, double* out, ct_stream_t stream) {
  if (!images || !axes || !out || n_views < 1 || rows < 1 || cols < 1)
    return set_err(CT_ERR_ARG, "bad strip-profile arguments");
  strip_profile_kernel<<<n_views, 256, 0, CT_STREAM(stream)>>>(images, rows, cols, axes, offset,
                                                               width, out);
  return check_launch("strip_profile_kernel");
}

}  // extern "C"
