// ct_bp.cu -- voxel-driven back-projection (_kernels.py:350-443) with the fused
// SART / OS-SART update (recon.py:105-119), and its footprint packing.
#include "ct_common.cuh"

#include <cuda.h>   // CUtensorMap (the TMA-staged BP variant, CT_BP_TMA)

namespace {

// TMA staging of the BP's footprint quads (A/B, run time CT_BP_TMA=1): per
// view pair, each CTA's detector window (the bounding box of its 64 x 4 voxel
// tile's footprints, from the tile's corner voxels) is brought into shared
// memory with cp.async.bulk.tensor (one box of TMA_BU x bv quads per view,
// mbarrier completion), and interior footprints inside the window read their
// quad from shared memory instead of global/L1.  Windows that do not fit the
// box, and footprints outside it, use the global path (same arithmetic).
#ifndef CT_BP_TMA_BU
#define CT_BP_TMA_BU 64
#endif
constexpr int TMA_BU = CT_BP_TMA_BU;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      " .reg .pred p;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// 4-D tile load (quads as FLOAT32 {4, cols, rows, n_batch}) into shared memory
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar,
                                            int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3),
      "r"(smem_u32(bar))
      : "memory");
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
#define CT_BP_UNROLL 8
#endif
constexpr int BP_UNROLL = CT_BP_UNROLL;
#ifndef CT_BP_MIN_BLOCKS
#define CT_BP_MIN_BLOCKS 8       // 32 registers, 64 warps/SM (A/B: 4-8)
#endif
constexpr int BP_MIN_BLOCKS = CT_BP_MIN_BLOCKS;
constexpr int BP_CHUNK = 64;   // views staged in shared memory per pass
static_assert(BP_CHUNK / 2 <= 32, "slow-pair mask is 32 bits");
constexpr float BP_EDGE_EPS = 1e-3f;  // px band around the frame edge refined in fp64
// Voxel patch per warp: BP_PR consecutive voxels along a row (r / x) times
// 32 / BP_PR consecutive rows (theta / y).  A compact patch projects onto
// fewer detector quads than a 32-voxel line (whose spread along u follows
// the line's extent across the view direction), so a warp's footprint loads
// touch fewer L1 sectors; mu I/O stays 32-byte sectors.  CTA = BP_THREADS/32
// warps side by side along the row.
#ifndef CT_BP_PR
#define CT_BP_PR 8
#endif
constexpr int BP_PR = CT_BP_PR, BP_PT = 32 / BP_PR;
constexpr int BP_SEG = BP_PR * (BP_THREADS / 32);   // row voxels per CTA
static_assert(32 % BP_PR == 0, "BP_PR");

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
  __host__ __device__ int row_len() const { return nr; }
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
  __host__ __device__ int row_len() const { return nx; }
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
  int vox_off, vox_end;   // voxels [vox_off, vox_end) (a rank's shard, distributed.py)
  int row0, nseg;         // first row of the range; CTAs per row group
  int tma_bv;             // TMA: window rows (box dim 2); the box is TMA_BU x tma_bv quads
  CUtensorMap tmap;       // TMA: the quads of the batch (CT_BP_TMA)
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
template <class Vox, int MODE, bool QUADS, bool TMA = false>
__global__ void __launch_bounds__(BP_THREADS, TMA ? 4 : BP_MIN_BLOCKS) bp_kernel(const __grid_constant__ BpArgs<Vox> a) {
  __shared__ BpPairF sv[BP_CHUNK / 2];
  // TMA: two windows (the views of a pair) in dynamic shared memory
  extern __shared__ __align__(128) float4 win[];
  __shared__ int2 worg[2];                 // window origin (u, v) per pair view; x = INT_MIN: none
  __shared__ __align__(8) uint64_t tbar;
  unsigned tphase = 0;
  if (TMA && threadIdx.x == 0) {
    mbar_init(&tbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  const int nr = a.vox.row_len();
  const int bs = (int)(blockIdx.x % (unsigned)a.nseg), bg = (int)(blockIdx.x / (unsigned)a.nseg);
  const int i = bs * BP_SEG + (threadIdx.x >> 5) * BP_PR + (threadIdx.x & (BP_PR - 1));
  const int q = a.row0 + bg * BP_PT + (threadIdx.x & 31) / BP_PR;
  const int m = q * nr + i;
  const bool active = i < nr && m >= a.vox_off && m < a.vox_end;
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
    if (!TMA && !active) continue;
    const float* __restrict__ img0 = a.corr + (size_t)c0 * npix;
    const int np = nc >> 1;
    unsigned slow = 0;   // pairs of this chunk for the slow path (BP_CHUNK / 2 <= 32)
#pragma unroll BP_UNROLL
    for (int i = 0; i < np; ++i) {
      const BpPairF f = sv[i];
      if (TMA) {
        // corner voxels of the CTA tile (2 row ends x 4 rows) projected into
        // both views of the pair: lanes 0-7 view 0, 8-15 view 1 of warp 0
        __syncthreads();                     // the previous pair's windows are consumed
        if (threadIdx.x < 32) {
          const int l = (threadIdx.x >> 3) & 1, cidx = threadIdx.x & 7;
          const int bs0 = (int)(blockIdx.x % (unsigned)a.nseg);
          const int bg0 = (int)(blockIdx.x / (unsigned)a.nseg);
          const int ci = min(bs0 * BP_SEG + (cidx & 1) * (BP_SEG - 1), nr - 1);
          const int cq = a.row0 + bg0 * BP_PT + (cidx >> 1);
          const long long cm = (long long)cq * nr + ci;
          float umin = 3.0e38f, umax = -3.0e38f, vmin = 3.0e38f, vmax = -3.0e38f;
          if (threadIdx.x < 16 && cm < a.vox.count()) {
            double w64[3];
            a.vox.world((int)cm, w64);
            const float* fp = reinterpret_cast<const float*>(&sv[i]);
            const float cphi = fp[0 + l], sphi = fp[2 + l], sod = fp[4 + l], sdd_p = fp[6 + l];
            const float u0 = fp[8 + l], v0 = fp[10 + l];
            const float xw0 = (float)w64[0], yw0 = (float)w64[1], zw0 = (float)w64[2];
            const float xi = fmaf(cphi, xw0, sphi * -yw0);
            const float depth = sod + fmaf(sphi, xw0, cphi * yw0);
            const float sc = sdd_p / depth;
            umin = umax = fmaf(xi, sc, u0) - 1.0f;   // u, v (the table holds u0 + 1, v0 + 1)
            vmin = vmax = fmaf(zw0, sc, v0) - 1.0f;
          }
          for (int o = 1; o < 8; o <<= 1) {
            umin = fminf(umin, __shfl_xor_sync(0xffffffffu, umin, o));
            umax = fmaxf(umax, __shfl_xor_sync(0xffffffffu, umax, o));
            vmin = fminf(vmin, __shfl_xor_sync(0xffffffffu, vmin, o));
            vmax = fmaxf(vmax, __shfl_xor_sync(0xffffffffu, vmax, o));
          }
          if (threadIdx.x == 0 || threadIdx.x == 8) {
            // 1 px slack each side (fp32 corners vs the voxels' own projections)
            const float ul = floorf(umin) - 1.0f, vl = floorf(vmin) - 1.0f;
            const bool fits = umin < 1.0e30f && floorf(umax) + 2.0f - ul < (float)TMA_BU &&
                              floorf(vmax) + 2.0f - vl < (float)a.tma_bv &&
                              fabsf(ul) < 1.0e6f && fabsf(vl) < 1.0e6f;
            worg[l] = fits ? make_int2((int)ul, (int)vl) : make_int2(INT_MIN, 0);
          }
        }
        __syncthreads();
        const int2 o0 = worg[0], o1 = worg[1];
        const bool s0 = o0.x != INT_MIN, s1 = o1.x != INT_MIN && 2 * i + 1 < nc;
        if (threadIdx.x == 0 && (s0 || s1)) {
          const unsigned box = (unsigned)(TMA_BU * a.tma_bv * 16);
          mbar_arrive_expect_tx(&tbar, box * ((s0 ? 1u : 0u) + (s1 ? 1u : 0u)));
          if (s0) tma_load_4d(win, &a.tmap, &tbar, 0, o0.x, o0.y, c0 + 2 * i);
          if (s1) tma_load_4d(win + TMA_BU * a.tma_bv, &a.tmap, &tbar, 0, o1.x, o1.y, c0 + 2 * i + 1);
        }
        if (s0 || s1) {
          mbar_wait(&tbar, tphase);
          tphase ^= 1u;
        }
        if (!active) continue;
      }
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
#if defined(CT_DEBUG_BOUNDS) && CT_DEBUG_BOUNDS
          assert((long long)oa < (long long)a.n_batch * npix &&
                 (long long)ob < (long long)a.n_batch * npix);
#endif
          // one 16-byte footprint per view; lerp-form bilinear per lane
          float4 qa, qb;
          if (TMA) {
            // quad (iv, iu) = floor bits - magic - 1 (U1 = u + 1), window-relative
            const int2 o0 = worg[0], o1 = worg[1];
            const int lua = (int)(tu.x - kMagicBits) - 1 - o0.x, lva = (int)(tv.x - kMagicBits) - 1 - o0.y;
            const int lub = (int)(tu.y - kMagicBits) - 1 - o1.x, lvb = (int)(tv.y - kMagicBits) - 1 - o1.y;
            const bool ina = o0.x != INT_MIN && (unsigned)lua < (unsigned)TMA_BU &&
                             (unsigned)lva < (unsigned)a.tma_bv;
            const bool inb = o1.x != INT_MIN && (unsigned)lub < (unsigned)TMA_BU &&
                             (unsigned)lvb < (unsigned)a.tma_bv;
            qa = ina ? win[lva * TMA_BU + lua] : ld_quad(a.quads + oa);
            qb = inb ? win[TMA_BU * a.tma_bv + lvb * TMA_BU + lub] : ld_quad(a.quads + ob);
          } else {
            qa = ld_quad(a.quads + oa);
            qb = ld_quad(a.quads + ob);
          }
          float fua, fub, fva, fvb;
          upk(FU, fua, fub);
          upk(FV, fva, fvb);
          // quad = (t00, t10 | t01, t11): the u-lerps of both rows are one
          // f32x2 subtract + one FFMA2 (the ops of the scalar lerps, lane for lane)
          float aa, ba, ab, bb;
          {
            const f32x2 P0 = pk(qa.x, qa.y), P1 = pk(qa.z, qa.w);
            upk(fma2(sub2(P1, P0), dup2(fua), P0), aa, ba);
          }
          {
            const f32x2 P0 = pk(qb.x, qb.y), P1 = pk(qb.z, qb.w);
            upk(fma2(sub2(P1, P0), dup2(fub), P0), ab, bb);
          }
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
      } else {
        slow |= 1u << i;   // deferred: keeps the slow path out of the hot loop
      }
    }
    // interior pairs: den += 1 per view, counted from the slow mask (no
    // per-pair counter in the hot loop)
    if (TMA && !active) continue;          // (after the pair loop's barriers)
    nfast += 2 * (np - __popc(slow));
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
      if (a.upd.n_peers > 0) {
        // all-gather of the updated shard fused into the update: every
        // rank's replica gets the voxel (NVLink peer stores); with
        // peer_ranges only the replicas whose range holds it (slab halos)
        for (int p = 0; p < a.upd.n_peers; ++p) {
          if (a.upd.peer_ranges && ((int64_t)m < __ldg(a.upd.peer_ranges + 2 * p) ||
                                    (int64_t)m >= __ldg(a.upd.peer_ranges + 2 * p + 1)))
            continue;
          a.upd.mu_peers[p][m] = mu;
        }
      } else {
        a.upd.mu[m] = mu;
      }
    }
  }
}

bool bp_tma_enabled() {
  const char* e = getenv("CT_BP_TMA");
  return e && e[0] == '1';
}
int bp_tma_rows() {
  const char* e = getenv("CT_BP_TMA_BV");
  const int v = e ? atoi(e) : 12;
  return v < 2 ? 2 : (v > 64 ? 64 : v);
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

// The batch's footprint quads [n_batch][rows][cols] float4 as a 4-D FLOAT32
// tensor {4, cols, rows, n_batch}; box {4, TMA_BU, bv, 1}; out-of-bounds
// elements (windows past the frame) read as zero.
int encode_quads_map(CUtensorMap* map, const float* quads, const ct_batch& b, int bv) {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&fn),
                                cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess || !fn)
      return set_err(CT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  }
  const cuuint64_t dims[4] = {4, (cuuint64_t)b.det_cols, (cuuint64_t)b.det_rows,
                              (cuuint64_t)b.n_batch};
  const cuuint64_t strides[3] = {16, 16ull * b.det_cols, 16ull * b.det_cols * b.det_rows};
  const cuuint32_t box[4] = {4, (cuuint32_t)TMA_BU, (cuuint32_t)bv, 1};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  const CUresult r = fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(quads), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? CT_OK : set_err(CT_ERR_CUDA, "cuTensorMapEncodeTiled failed");
}

template <class Vox, int MODE>
int launch_bp(const Vox& vox, const float* corr, const float* quads, const ct_det_view* dets,
              const ct_batch& b, float* num, float* den, const ct_update* upd, cudaStream_t st,
              int64_t offset = 0, int64_t count = -1) {
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
  const int64_t nvox = count < 0 ? vox.count() : count;
  a.vox_off = (int)offset;
  a.vox_end = (int)(offset + nvox);
  if (nvox == 0) return CT_OK;
  const int nr = vox.row_len();
  const int64_t row0 = offset / nr, row_end = (offset + nvox + nr - 1) / nr;
  a.row0 = (int)row0;
  a.nseg = (nr + BP_SEG - 1) / BP_SEG;
  const int64_t groups = (row_end - row0 + BP_PT - 1) / BP_PT;
  const unsigned blocks = (unsigned)(groups * a.nseg);
  if (MODE == BP_UPDATE && quads && bp_tma_enabled()) {
    a.tma_bv = bp_tma_rows();
    int rc = encode_quads_map(&a.tmap, quads, b, a.tma_bv);
    if (rc) return rc;
    const int smem = 2 * TMA_BU * a.tma_bv * 16;
    static bool attr_set = false;
    if (!attr_set) {
      cudaFuncSetAttribute(bp_kernel<Vox, MODE, true, true>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
      attr_set = true;
    }
    bp_kernel<Vox, MODE, true, true><<<blocks, BP_THREADS, smem, st>>>(a);
    return check_launch("bp_kernel (TMA)");
  }
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

// bilinear footprints of a correction stack: quad (v, u) = (c[v][u], c[v+1][u],
// c[v][u+1], c[v+1][u+1]) of the same image (column pairs, so the BP's two
// u-lerps are one f32x2 op), 0 past the last row / column (never read: the
// BP's fast path only takes footprints inside the frame)
__global__ void pack_quads_kernel(const float* __restrict__ corr, int64_t n, int rows, int cols,
                                  float4* __restrict__ quads) {
  const int64_t m = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= n) return;
  const int u = (int)(m % cols), v = (int)((m / cols) % rows);
  const bool ru = u + 1 < cols, rv = v + 1 < rows;
  const float* p = corr + m;
  quads[m] = make_float4(__ldg(p), rv ? __ldg(p + cols) : 0.0f, ru ? __ldg(p + 1) : 0.0f,
                         (ru && rv) ? __ldg(p + cols + 1) : 0.0f);
}


}  // namespace

extern "C" {

static int check_bp(const float* corr, const ct_det_view* dets, const ct_batch* b) {
  if (!corr || !dets || !b) return set_err(CT_ERR_ARG, "null corr/dets/batch");
  if (b->n_batch < 1 || b->det_rows < 1 || b->det_cols < 1)
    return set_err(CT_ERR_ARG, "bad batch dimensions");
  // the BP addresses the correction stack with 32-bit element offsets
  if ((int64_t)b->n_batch * b->det_rows * b->det_cols > (int64_t)0xFFFFFFFFu)
    return set_err(CT_ERR_ARG, "BP batch too large (n_batch*rows*cols must be < 2^32)");
  return CT_OK;
}

// every entry point that takes a ct_update: mu present, and a consistent peer
// list (n_peers >= 0; n_peers > 0 needs the device pointer array)
static int check_update(const ct_update* upd) {
  if (!upd || !upd->mu) return set_err(CT_ERR_ARG, "null update/mu");
  if (upd->n_peers < 0 || (upd->n_peers > 0 && !upd->mu_peers))
    return set_err(CT_ERR_ARG, "bad update peer list");
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
  if (!trig) return set_err(CT_ERR_ARG, "null trig");
  if ((rc = check_update(upd))) return rc;
  CylVox vox;
  vox.init(*grid, trig);
  return launch_bp<CylVox, BP_UPDATE>(vox, corr, quads, dets, *batch, nullptr, nullptr, upd,
                                      CT_STREAM(stream));
}

int ct_bp_cart_update(const float* corr, const float* quads, const ct_det_view* dets, const ct_batch* batch,
                      const ct_cart_grid* grid, const ct_update* upd, ct_stream_t stream) {
  int rc = check_bp(corr, dets, batch);
  if (rc || (rc = check_cart(grid))) return rc;
  if ((rc = check_update(upd))) return rc;
  CartVox vox;
  vox.init(*grid);
  return launch_bp<CartVox, BP_UPDATE>(vox, corr, quads, dets, *batch, nullptr, nullptr, upd,
                                       CT_STREAM(stream));
}

int ct_bp_cyl_update_range(const float* corr, const float* quads, const ct_det_view* dets,
                           const ct_batch* batch, const ct_cyl_grid* grid, const double* trig,
                           const ct_update* upd, int64_t offset, int64_t count,
                           ct_stream_t stream) {
  int rc = check_bp(corr, dets, batch);
  if (rc || (rc = check_cyl(grid))) return rc;
  if (!trig) return set_err(CT_ERR_ARG, "null trig");
  if ((rc = check_update(upd))) return rc;
  const int64_t n = (int64_t)grid->n_h * grid->n_theta * grid->n_r;
  if (offset < 0 || count < 0 || offset + count > n) return set_err(CT_ERR_ARG, "bad voxel range");
  CylVox vox;
  vox.init(*grid, trig);
  return launch_bp<CylVox, BP_UPDATE>(vox, corr, quads, dets, *batch, nullptr, nullptr, upd,
                                      CT_STREAM(stream), offset, count);
}

int ct_bp_cart_update_range(const float* corr, const float* quads, const ct_det_view* dets,
                            const ct_batch* batch, const ct_cart_grid* grid, const ct_update* upd,
                            int64_t offset, int64_t count, ct_stream_t stream) {
  int rc = check_bp(corr, dets, batch);
  if (rc || (rc = check_cart(grid))) return rc;
  if ((rc = check_update(upd))) return rc;
  const int64_t n = (int64_t)grid->n_z * grid->n_y * grid->n_x;
  if (offset < 0 || count < 0 || offset + count > n) return set_err(CT_ERR_ARG, "bad voxel range");
  CartVox vox;
  vox.init(*grid);
  return launch_bp<CartVox, BP_UPDATE>(vox, corr, quads, dets, *batch, nullptr, nullptr, upd,
                                       CT_STREAM(stream), offset, count);
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
  // the stand-alone update writes mu only (peer replicas: the fused BP update)
  if (upd->n_peers != 0) return set_err(CT_ERR_ARG, "ct_sart_update does not take peer replicas");
  if (count == 0) return CT_OK;
  update_kernel<<<blocks_for(count, 256), 256, 0, CT_STREAM(stream)>>>(num, den, offset, count,
                                                                       *upd);
  return check_launch("update_kernel");
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

}  // extern "C"
