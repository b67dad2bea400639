// ct_fp.cu -- forward projection (_kernels.py:238-343): ray march, correction /
// residual / row-sum epilogues, and the volume gather layouts it reads.
#include "ct_common.cuh"

namespace {

// ---------------------------------------------------------------------------
// forward projection
// ---------------------------------------------------------------------------
// EPI_CORR_RESID: the correction epilogue plus residual partials -- the
// residual FP of pass k and the first subset's correction FP of pass k+1 read
// the same mu, so one march serves both (recon.SartRun)
// EPI_ROWCOUNT: in-support samples summed per detector row (no march; the
// per-row cost model of the angle-sharded row split, distributed.py)
enum FpEpi { EPI_PROJECT = 0, EPI_CORR = 1, EPI_RESID = 2, EPI_ROWMAX = 3, EPI_CORR_RESID = 4,
             EPI_ROWCOUNT = 5 };

// FP volume layouts: plain mu, the 32-byte polynomial cells (ct_pack_gather_*),
// or 16-byte corner quads per h layer (large volumes; see gather_quad())
// GL_OCTB: the 32-byte cells in 2x2 (row, column) bricks per 128-byte line, for
// volumes whose layers exceed the small-layer bound (A/B: C4-cart FP -6 %; C2 +15 %)
enum FpLayout { GL_PLAIN = 0, GL_OCT = 1, GL_QUAD = 2, GL_OCTB = 3 };

// block = FP_WX x FP_WY warps, each warp a pixel patch (tile_ww x tile_wh rays)
#ifndef CT_DEBUG_BOUNDS
#define CT_DEBUG_BOUNDS 0        // device asserts on every gather-layout cell address (tests)
#endif
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
// GL_OCT volumes whose 32-byte-cell layers fit well inside L2 (<= 6 MB: C1-C3)
// run a 56-register variant (36 warps/SM; A/B C2 -1.1 %); larger ones (C4-cart)
// lose 3 % with it, the GL_QUAD path 11 % (C5)
#ifndef CT_FP_MAXREG_SMALL
#define CT_FP_MAXREG_SMALL 56
#endif
#ifndef CT_FP_WW1
#define CT_FP_WW1 4              // warp patch width at one lane per ray
#endif
// Depth-aligned march (A/B only, rejected): the lanes of a warp step through
// their samples in lockstep by depth along the view direction instead of by
// their own sample index, so that at every step the warp's 32 samples lie
// near one plane across the rays -- the hypothesis being fewer distinct
// 128-byte lines per quarter-warp load (L1TEX data-pipe wavefronts: one per
// distinct line per 8 lanes, tools/microbench/l1_wavefronts.cu).  Measured
// (C5 correction FP, ncu): 8.16 wavefronts per request either way (the lanes'
// cells are one pixel apart, not misaligned in depth), +10 % instructions for
// the per-sample validity: C5 0.276 -> 0.289 s (1 chain, =2) / 0.316 s (2
// chains, =1), C2 192 -> 227 / 237 ms.
#ifndef CT_FP_ALIGN
#define CT_FP_ALIGN 0
#endif
// CT_QUAD_TEX (A/B): GL_QUAD cell loads through the texture pipe (a linear
// float4 texture over the gather buffer) instead of LSU global loads -- 1: the
// second layer of a cell only (splits the loads across the two L1TEX input
// pipes), 2: both layers
#ifndef CT_QUAD_TEX
#define CT_QUAD_TEX 0
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
  // residual partial slots: 0 -> block (x, b, z) writes partial
  // (z * gridDim.y + b) * gridDim.x + x; > 0 -> (z * red_rows + view_ids[b]) *
  // gridDim.x + x, i.e. the slot of the view in an identity-ordered batch of
  // red_rows views, so launches over disjoint view sets fill one scratch whose
  // fixed-order sum equals the single launch's bit for bit
  int red_rows;
  // flattened-row range (angle sharding, distributed.py): only rays of rows
  // f = b * rows + row in [frow_lo, frow_hi) are marched, and the correction
  // of row f lands at out0[(f - frow_lo) * cols + col].  Defaults: all rows.
  int64_t frow_lo, frow_hi;
  // peer-store all-gather of the corrections (distributed.py, fused comm):
  // with n_peers > 0 every correction goes to peers[p][peer_off + out index]
  float* const* __restrict__ peers;
  int n_peers;
  int64_t peer_off;
  // per-view detector-row bands (slab decomposition, distributed.SlabSartRun):
  // with bands set, view slot b marches rows [bands[2b], bands[2b+1]) only,
  // grid z counting row tiles from bands[2b] (a multiple of the row tile, so
  // residual partial slots stay those of the full launch); outputs land at
  // their full-stack positions (frow_lo = 0)
  const int32_t* __restrict__ bands;
  // per-peer row ranges of the peer stores (slab decomposition, fused): with
  // peer_rows set, view slot b's row `row` goes to peer p only when
  // peer_rows[2 (b n_peers + p)] <= row < peer_rows[2 (b n_peers + p) + 1]
  const int32_t* __restrict__ peer_rows;
};

// A correction value: local output, or (fused all-gather) every rank's copy
// of the gathered stack over NVLink peer stores.
template <class Geo>
__device__ __forceinline__ void store_corr(const FpArgs<Geo>& a, size_t oidx, float c, int b,
                                           int row) {
  if (a.n_peers > 0) {
    for (int p = 0; p < a.n_peers; ++p) {
      if (a.peer_rows) {
        const int* r = a.peer_rows + 2 * ((size_t)b * a.n_peers + p);
        if (row < __ldg(r) || row >= __ldg(r + 1)) continue;
      }
      a.peers[p][a.peer_off + (int64_t)oidx] = c;
    }
  } else {
    a.out0[oidx] = c;
  }
}

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
    unsigned prev = 0x80000000u;   // no cell (indices are >= -1, or >= B - 1 < 2^31)
    float4 pa = make_float4(0.f, 0.f, 0.f, 0.f), pb = make_float4(0.f, 0.f, 0.f, 0.f);
    float sum = 0.0f;
  };
  auto value = [&](Chain& ch, const Cell& c) -> float {
    if (OCT == GL_OCTB) {
      const unsigned idx = geo.template oct_cell<WRAP>(c);
#if CT_DEBUG_BOUNDS
      assert(8LL * ((long long)idx + 1) <= geo.dbg_floats);
#endif
      if (idx != ch.prev) ld_cell(geo.qraw + 2 * (size_t)idx, ch.pa, ch.pb);
      ch.prev = idx;
      return trilinear_eval(ch.pa, ch.pb, c.w0, c.w1, c.w2);
    }
    if (OCT == GL_OCT) {
      const unsigned idx = geo.template gather_index<WRAP>(c);
#if CT_DEBUG_BOUNDS
      {
        const long long cell = (long long)(geo.oct - geo.qraw) / 2 + cell_off(idx);
        assert(cell >= 0 && 8LL * (cell + 1) <= geo.dbg_floats);
      }
#endif
      // signed: the cylindrical r bits make the first cell's index -1 (kRMagic)
      if (idx != ch.prev) ld_cell(geo.oct + 2 * cell_off(idx), ch.pa, ch.pb);
      ch.prev = idx;   // (unconditional: equal when not reloaded; no predicated move)
      return trilinear_eval(ch.pa, ch.pb, c.w0, c.w1, c.w2);
    }
    if (OCT == GL_QUAD) {
      // bilinear layers k, k+1 of the cell; the h terms are their
      // difference (two f32x2 subtractions)
#if CT_QUAD_BRICK
      const unsigned idx = geo.template quad_cell<WRAP>(c, 0u);
#if CT_DEBUG_BOUNDS
      assert(geo.quad_cell_up(c, idx) == geo.template quad_cell<WRAP>(c, 1u));
      assert(4LL * ((long long)geo.template quad_cell<WRAP>(c, 1u) + 1) <= geo.dbg_floats &&
             4LL * ((long long)idx + 1) <= geo.dbg_floats);
#endif
      if (idx != ch.prev) {
#if CT_QUAD_TEX >= 2
        const float4 a = tex1Dfetch<float4>(geo.qtex, (int)idx);
#else
        const float4 a = ld_vquad(geo.qraw + idx);
#endif
#if CT_QUAD_TEX >= 1
        const float4 b = tex1Dfetch<float4>(geo.qtex, (int)geo.quad_cell_up(c, idx));
#else
        const float4 b = ld_vquad(geo.qraw + geo.quad_cell_up(c, idx));
#endif
#else
      const unsigned idx = geo.template gather_index<WRAP>(c);
      if (idx != ch.prev) {
        const float4 a = ld_vquad(geo.oct + cell_off(idx));
        const float4 b = ld_vquad(geo.oct + cell_off(idx) + geo.cell_kstride);
#endif
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

// Depth-aligned march of the interior samples [0, n_int) of a ray whose
// first sample has global depth index D (CT_FP_ALIGN): the warp's depth range
// [G0, G1) is split at Gm into two chains marched in lockstep (chain 0 covers
// depths [G0, Gm), chain 1 [Gm, G1)); at iteration j chain c of this lane
// holds its sample k = base_c - D + j, valid when 0 <= k < end_c.  Cells are
// loaded only for valid samples that leave the chain's live cell; invalid
// samples contribute nothing.  + the last sample k_last when with_last.
template <class Geo, int OCT, bool WRAP>
__device__ __forceinline__ float march_aligned(const Geo& geo, const RayF& ry, int D, int n_int,
                                               int G0, int G1, bool with_last, float k_last) {
  struct Chain {
    unsigned prev = 0x80000000u;
    float4 pa = make_float4(0.f, 0.f, 0.f, 0.f), pb = make_float4(0.f, 0.f, 0.f, 0.f);
    float sum = 0.0f;
  };
  auto value = [&](Chain& ch, const Cell& c, bool valid) -> float {
    unsigned idx;
    if (OCT == GL_OCTB) {
      idx = geo.template oct_cell<WRAP>(c);
      if (valid && idx != ch.prev) ld_cell(geo.qraw + 2 * (size_t)idx, ch.pa, ch.pb);
    } else if (OCT == GL_OCT) {
      idx = geo.template gather_index<WRAP>(c);
      if (valid && idx != ch.prev) ld_cell(geo.oct + 2 * cell_off(idx), ch.pa, ch.pb);
    } else if (OCT == GL_PLAIN) {
      // the same 8 values from mu, coefficients in-kernel (identical bits)
      idx = 0u;
      if (valid) {
        float4 a, b;
        geo.fetch_plain(c, a, b);
        trilinear_coeffs(a, b, ch.pa, ch.pb);
      }
      return trilinear_eval(ch.pa, ch.pb, c.w0, c.w1, c.w2);
    } else {
      idx = geo.template quad_cell<WRAP>(c, 0u);
      if (valid && idx != ch.prev) {
        const float4 a = ld_vquad(geo.qraw + idx);
        const float4 b = ld_vquad(geo.qraw + geo.quad_cell_up(c, idx));
        ch.pa = a;
        float x0, x1, y0, y1;
        upk(sub2(pk(b.x, b.y), pk(a.x, a.y)), x0, x1);
        upk(sub2(pk(b.z, b.w), pk(a.z, a.w)), y0, y1);
        ch.pb = make_float4(x0, x1, y0, y1);
      }
    }
    ch.prev = valid ? idx : ch.prev;
    return trilinear_eval(ch.pa, ch.pb, c.w0, c.w1, c.w2);
  };
#if CT_FP_ALIGN == 2
  // one chain: two consecutive samples per f32x2 locate
  Chain ch;
  const int T = G1 - G0;                        // <= 0: no interior samples in the warp
  int k = G0 - D;
  const unsigned e = (unsigned)n_int;
  f32x2 KF = pk((float)k, (float)(k + 1));
#pragma unroll FP_UNROLL
  for (int j = 0; j < T; j += 2) {
    Cell c0, c1;
    geo.locate2(KF, ry, c0, c1);
    KF = add2(KF, dup2(2.0f));
    const bool v0 = (unsigned)k < e, v1 = (unsigned)(k + 1) < e;
    k += 2;
    const float a0 = value(ch, c0, v0);
    const float a1 = value(ch, c1, v1);
    ch.sum += (v0 ? a0 : 0.0f) + (v1 ? a1 : 0.0f);
  }
  float sum = ch.sum;
  if (with_last) sum += value(ch, geo.locate1(k_last, ry), true);
  return sum;
#else
  Chain ch0, ch1;
  // G0 > G1: no lane of the warp has interior samples
  const int Gm = G1 >= G0 ? G0 + (G1 - G0 + 1) / 2 : G0;
  const int T = Gm - G0;                        // >= G1 - Gm
  int k0 = G0 - D;                              // chain 0's sample; chain 1's is k0 + T
  const unsigned e0 = (unsigned)max(0, min(n_int, Gm - D)), e1 = (unsigned)n_int;
  f32x2 KF = pk((float)k0, (float)(k0 + T));
#pragma unroll FP_UNROLL
  for (int j = 0; j < T; j += 2) {
    Cell c0, c1, c2, c3;
    geo.locate2(KF, ry, c0, c1);
    geo.locate2(add2(KF, dup2(1.0f)), ry, c2, c3);
    KF = add2(KF, dup2(2.0f));
    // (unsigned)k < end: 0 <= k < end in one compare
    const int k1 = k0 + T;
    const bool v0 = (unsigned)k0 < e0, v1 = (unsigned)k1 < e1;
    const bool v2 = (unsigned)(k0 + 1) < e0, v3 = (unsigned)(k1 + 1) < e1;
    k0 += 2;
    const float a0 = value(ch0, c0, v0);
    const float b0 = value(ch1, c1, v1);
    const float a1 = value(ch0, c2, v2);
    const float b1 = value(ch1, c3, v3);
    ch0.sum += (v0 ? a0 : 0.0f) + (v2 ? a1 : 0.0f);
    ch1.sum += (v1 ? b0 : 0.0f) + (v3 ? b1 : 0.0f);
  }
  float sum = ch0.sum + ch1.sum;
  if (with_last) sum += value(ch1, geo.locate1(k_last, ry), true);
  return sum;
#endif
}

// One sub-ray, chunk `chunk` of `K`: returns this chunk's in-support sample
// count and adds the fp32 sum of its interpolated values into acc (COUNT_ONLY:
// chunk 0 returns the whole ray's count, without marching).
template <class Geo, bool NEAREST, int OCT, bool COUNT_ONLY>
__device__ __forceinline__ int march(const Geo& geo, const ct_ray_view& v, double cu, double cv,
                                     double step, float& acc, int chunk, int K, bool present) {
  // ALIGNED: every lane of the warp arrives here (present or not) -- the
  // warp's depth range is a full-warp reduction
  constexpr bool ALIGNED = CT_FP_ALIGN && !NEAREST && !COUNT_ONLY;
  const bool aligned = ALIGNED && K == 1;
  double d[3];
  double t0 = 0.0, t1 = 0.0;
  bool hit = false;
  if (present) {
    subray_dir(v, cu, cv, d);
    hit = geo.interval(v.src, d, t0, t1) && t1 > t0;
  }
  int n = 0;
  if (hit) n = (int)ceil(ddiv(dsub(t1, t0), step));
  int G0 = 0, G1 = 0, D = 0;
  if (aligned) {
    D = hit ? (int)floor(ddiv(t0, step)) : 0;     // depth index of the ray's first sample
    const bool interior = hit && n > 1;
    G0 = __reduce_min_sync(0xffffffffu, interior ? D : INT_MAX);
    G1 = __reduce_max_sync(0xffffffffu, interior ? D + n - 1 : INT_MIN);
  }
  if (!hit) return 0;
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
  const bool wrap = __any_sync(__activemask(), ry.wrap);
  if (ALIGNED && aligned) {
    if (wrap)
      sum = march_aligned<Geo, OCT, true>(geo, ry, D, n_int, G0, G1, with_last, (float)n_int);
    else
      sum = march_aligned<Geo, OCT, false>(geo, ry, D, n_int, G0, G1, with_last, (float)n_int);
  } else if (wrap) {
    sum = march_linear<Geo, OCT, true>(geo, ry, k, k_end, with_last, (float)n_int);
  } else {
    sum = march_linear<Geo, OCT, false>(geo, ry, k, k_end, with_last, (float)n_int);
  }
  acc += sum;
  return (k_end - (chunk * n_int) / K) + ((own_last && last_in) ? 1 : 0);
}


template <class Geo, int EPI, bool NEAREST, int OCT>
__device__ __forceinline__ void fp_body(const FpArgs<Geo>& a);

template <class Geo, int EPI, bool NEAREST, int OCT>
__global__ void __maxnreg__(CT_FP_MAXREG) fp_kernel(const FpArgs<Geo> a) {
  fp_body<Geo, EPI, NEAREST, OCT>(a);
}

// the same kernel under the small-volume register cap (see CT_FP_MAXREG_SMALL)
template <class Geo, int EPI, bool NEAREST, int OCT>
__global__ void __maxnreg__(CT_FP_MAXREG_SMALL) fp_kernel_small(const FpArgs<Geo> a) {
  fp_body<Geo, EPI, NEAREST, OCT>(a);
}

// Thread / block indices read through volatile asm: the epilogue re-derives
// the pixel instead of keeping it live across the march (ptxas otherwise
// spills the pixel's 64-bit offsets to local memory once per ray, ~40 B/ray
// of write-back traffic that ends in DRAM -- 0.46 GB per C2 correction launch)
__device__ __forceinline__ unsigned vol_tid() {
  unsigned r;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint3 vol_ctaid() {
  uint3 r;
  asm volatile("mov.u32 %0, %%ctaid.x;" : "=r"(r.x));
  asm volatile("mov.u32 %0, %%ctaid.y;" : "=r"(r.y));
  asm volatile("mov.u32 %0, %%ctaid.z;" : "=r"(r.z));
  return r;
}
__host__ __device__ inline int ilog2_small(int x) { return x >= 8 ? 3 : x >= 4 ? 2 : x >= 2 ? 1 : 0; }

struct FpPixel {
  int lane, warp, chunk, col, row, b;
  bool active;
};
template <class Geo>
__device__ __forceinline__ FpPixel fp_pixel(const FpArgs<Geo>& a) {
  FpPixel p;
  const unsigned t = vol_tid();
  const uint3 blk = vol_ctaid();
  p.lane = t & 31;
  p.warp = t >> 5;
  const int K = a.lanes;                      // 1, 2, 4 or 8 (lanes_for)
  const int lk = ilog2_small(K);
  const int ww = tile_ww(K), wh = tile_wh(K), lw = ilog2_small(ww);
  p.chunk = p.lane & (K - 1);
  const int rslot = p.lane >> lk;
  // each warp covers a ww x wh pixel patch, the block FP_WX x FP_WY warps
  p.col = blk.x * (FP_WX * ww) + (p.warp % FP_WX) * ww + (rslot & (ww - 1));
  p.row = blk.z * (FP_WY * wh) + (p.warp / FP_WX) * wh + (rslot >> lw);
  p.b = blk.y;
  if (a.bands) {
    const int lo = __ldg(a.bands + 2 * p.b), hi = min(__ldg(a.bands + 2 * p.b + 1), a.rows);
    p.row += lo;
    p.active = p.row < hi && p.col < a.cols;
    return p;
  }
  const int64_t frow = (int64_t)p.b * a.rows + p.row;
  p.active = p.row < a.rows && p.col < a.cols && frow >= a.frow_lo && frow < a.frow_hi;
  return p;
}

template <class Geo, int EPI, bool NEAREST, int OCT>
__device__ __forceinline__ void fp_body(const FpArgs<Geo>& a) {
  const int K = a.lanes;
  float acc = 0.0f;
  int count = 0;
  {
  const FpPixel p = fp_pixel(a);
  const int col = p.col, row = p.row, chunk = p.chunk;
  const bool active = p.active;
  const int vid = a.view_ids ? a.view_ids[p.b] : p.b;
  // every lane calls march (the depth-aligned march reduces over the whole
  // warp); lanes off the detector or outside the row range march nothing.
  // Row ranges are FP tile aligned (ct_fp_row_tile), i.e. whole warps.
  if (a.ss == 1) {
    // one sub-ray at the pixel centre ((0 + .5)/1 - .5 = 0 exactly): the view
    // basis is dead after the per-ray setup, keeping the march loop's
    // register footprint small
    count = march<Geo, NEAREST, OCT, EPI == EPI_ROWMAX || EPI == EPI_ROWCOUNT>(
        a.geo, a.views[active ? vid : 0], (double)col, (double)row, a.step, acc, chunk, K,
        active);
  } else {
    const ct_ray_view& v = a.views[active ? vid : 0];
    const int ss = a.ss;
    for (int sv = 0; sv < ss; ++sv) {
      const double off_v = dsub(ddiv((double)sv + 0.5, (double)ss), 0.5);
      for (int su = 0; su < ss; ++su) {
        const double off_u = dsub(ddiv((double)su + 0.5, (double)ss), 0.5);
        count += march<Geo, NEAREST, OCT, EPI == EPI_ROWMAX || EPI == EPI_ROWCOUNT>(
            a.geo, v, dadd((double)col, off_u), dadd((double)row, off_v), a.step, acc, chunk, K,
            active);
      }
    }
  }
  }
  // only acc / count crossed the march: the pixel is derived again
  const FpPixel p = fp_pixel(a);
  const int lane = p.lane, warp = p.warp, chunk = p.chunk, row = p.row, b = p.b;
  const bool active = p.active;
  const size_t npix = (size_t)a.rows * a.cols;
  const size_t pix = (size_t)row * a.cols + p.col;
  const size_t oidx = (size_t)b * npix + pix - (size_t)a.frow_lo * a.cols;   // out0 element
  const int vid = a.view_ids ? a.view_ids[b] : b;
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
  } else if (EPI == EPI_ROWCOUNT) {
    if (active && lead && count > 0)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.red) + (size_t)b * a.rows + row,
                (unsigned long long)count);
  } else if (EPI == EPI_CORR) {
    if (active && lead) {
      float c = 0.0f;
      if (w64 > a.row_thr[vid]) {
        const float pm = a.p_meas[(size_t)vid * npix + pix];
        c = (pm - (float)p64) / (float)w64;
      }
      store_corr(a, oidx, c, b, row);
    }
  } else {
    double x = 0.0;
    if (active && lead) {
      if (EPI == EPI_CORR_RESID) {
        // both epilogues from one read of p_meas, with the same ops as
        // EPI_CORR and EPI_RESID
        const float pm = a.p_meas[(size_t)vid * npix + pix];
        float c = 0.0f;
        if (w64 > a.row_thr[vid]) c = (pm - (float)p64) / (float)w64;
        store_corr(a, oidx, c, b, row);
        const double r = (double)pm - (double)(float)p64;
        x = r * r;
      } else if (EPI == EPI_RESID) {
        // compare with the fp32 simulation, i.e. what a stored projection of
        // this volume holds: consistent data gives exactly 0, as in the reference
        const double r = (double)a.p_meas[(size_t)vid * npix + pix] - (double)(float)p64;
        x = r * r;
      } else {
        x = w64;
      }
    }
    constexpr bool SUM = EPI == EPI_RESID || EPI == EPI_CORR_RESID;
    __shared__ double sred[FP_THREADS / 32];
    x = SUM ? warp_sum(x) : warp_max(x);
    if (lane == 0) sred[warp] = x;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = sred[0];
      for (int w = 1; w < FP_THREADS / 32; ++w)
        t = SUM ? t + sred[w] : fmax(t, sred[w]);
      if (SUM) {
        // the block's row tile in the full launch (band launches start at bands[2b])
        const unsigned zt = blockIdx.z + (a.bands ? (unsigned)__ldg(a.bands + 2 * b) /
                                                        (unsigned)(FP_WY * tile_wh(K))
                                                  : 0u);
        const size_t blk = a.red_rows > 0
            ? ((size_t)zt * a.red_rows + vid) * gridDim.x + blockIdx.x
            : ((size_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        // a band launch's tiles past this view's band (its grid spans the
        // longest band) hold another band's slots: no write
        const bool mine = !a.bands || (int)(zt * (unsigned)(FP_WY * tile_wh(K))) <
                                          __ldg(a.bands + 2 * b + 1);
        if (mine) a.red[blk] = t;
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

int fp_tile_rows(const ct_batch& b) {
  return FP_WY * tile_wh(lanes_for(b.det_rows, b.det_cols));
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

#if CT_DEBUG_BOUNDS || CT_QUAD_TEX
int64_t gather_floats_cyl(const ct_cyl_grid& g);
int64_t gather_floats_cart(const ct_cart_grid& g);
inline int64_t gather_floats_of(const CylGeo& g) {
  ct_cyl_grid c{};
  c.n_h = g.nh; c.n_theta = g.nt; c.n_r = g.nr;
  return gather_floats_cyl(c);
}
inline int64_t gather_floats_of(const CartGeo& g) {
  ct_cart_grid c{};
  c.n_z = g.nz; c.n_y = g.ny; c.n_x = g.nx;
  return gather_floats_cart(c);
}
#endif

template <class Geo, int EPI>
int launch_fp(const Geo& geo, const ct_ray_view* views, const ct_batch& b, const ct_sampling& s,
              const float* p_meas, const double* thr, float* o0, float* o1, double* red,
              cudaStream_t st, int red_rows = 0, int64_t frow_lo = 0,
              int64_t frow_hi = INT64_MAX, float* const* peers = nullptr, int n_peers = 0,
              int64_t peer_off = 0, const int32_t* bands = nullptr, int band_rows = 0,
              const int32_t* peer_rows = nullptr) {
  FpArgs<Geo> a;
  a.bands = bands;
  a.peer_rows = peer_rows;
  dim3 grid = fp_grid(b);
  if (bands) grid.z = (band_rows + fp_tile_rows(b) - 1) / fp_tile_rows(b);
  a.peers = peers;
  a.n_peers = n_peers;
  a.peer_off = peer_off;
#if CT_DEBUG_BOUNDS
  a.geo = geo;
  a.geo.dbg_floats = gather_floats_of(geo);
#endif
  a.red_rows = red_rows;
  a.frow_lo = frow_lo;
  a.frow_hi = frow_hi;
#if !CT_DEBUG_BOUNDS
  a.geo = geo;
#endif
#if CT_QUAD_TEX
  if (geo.quad && geo.qraw) {
    // one texture object per gather buffer, kept for the process lifetime
    static const void* tex_ptr[8] = {};
    static unsigned long long tex_obj[8] = {};
    static int tex_n = 0;
    int slot = -1;
    for (int i = 0; i < tex_n; ++i)
      if (tex_ptr[i] == geo.qraw) slot = i;
    if (slot < 0) {
      cudaResourceDesc rd = {};
      rd.resType = cudaResourceTypeLinear;
      rd.res.linear.devPtr = const_cast<float4*>(geo.qraw);
      rd.res.linear.desc = cudaCreateChannelDesc<float4>();
      rd.res.linear.sizeInBytes = (size_t)gather_floats_of(geo) * 4;
      cudaTextureDesc td = {};
      td.readMode = cudaReadModeElementType;
      td.filterMode = cudaFilterModePoint;
      cudaTextureObject_t t = 0;
      if (cudaCreateTextureObject(&t, &rd, &td, nullptr) != cudaSuccess)
        return check_launch("cudaCreateTextureObject");
      slot = tex_n < 8 ? tex_n++ : 7;
      tex_ptr[slot] = geo.qraw;
      tex_obj[slot] = t;
    }
    a.geo.qtex = tex_obj[slot];
  }
#endif
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
    fp_kernel<Geo, EPI, true, GL_PLAIN><<<grid, FP_THREADS, 0, st>>>(a);
  else if (EPI != EPI_ROWMAX && EPI != EPI_ROWCOUNT && geo.oct && geo.quad)
    fp_kernel<Geo, EPI, false, GL_QUAD><<<grid, FP_THREADS, 0, st>>>(a);
  else if (EPI != EPI_ROWMAX && EPI != EPI_ROWCOUNT && geo.oct && geo.obrick)
    fp_kernel<Geo, EPI, false, GL_OCTB><<<grid, FP_THREADS, 0, st>>>(a);
  else if (EPI != EPI_ROWMAX && EPI != EPI_ROWCOUNT && geo.oct)
  {
    if (32.0 * geo.cells_layer <= CT_FP_SMALL_LAYER_BYTES)
      fp_kernel_small<Geo, EPI, false, GL_OCT><<<grid, FP_THREADS, 0, st>>>(a);
    else
      fp_kernel<Geo, EPI, false, GL_OCT><<<grid, FP_THREADS, 0, st>>>(a);
  }
  else
    fp_kernel<Geo, EPI, false, GL_PLAIN><<<grid, FP_THREADS, 0, st>>>(a);
  return check_launch("fp_kernel");
}

// ---------------------------------------------------------------------------
// gather layout: cell m holds the trilinear polynomial coefficients of its
// 2x2x2 neighbourhood (r/h or x/y/z clamp, theta wrap) as two float4 = one
// 32-byte sector, so one FP sample is one 256-bit load instead of 8 scattered
// loads.
// ---------------------------------------------------------------------------
// one h-layer (blockIdx.y = kc) per grid row; cells past the layer's rows are
// the stride padding (zeroed, never read)
template <bool BRICK>
__global__ void pack_gather_cyl_kernel(const float* __restrict__ mu, int nh, int nt, int nr,
                                       unsigned ks, unsigned js, float4* __restrict__ oct, int kc0) {
  // cells (kc, jc, ic), kc in [0, nh], jc in [0, nt], ic in [0, nr]: corner
  // (kc-1, jc-1, ic-1); index -1 is a halo (r/h: copy of 0; theta: row nt-1).
  // Only real cells are written (the stride padding is never read).
  const unsigned rem = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned nc = (unsigned)nr + 1u;
  if (rem >= (unsigned)(nt + 1) * nc) return;
  const int kc = kc0 + (int)blockIdx.y;
  const int jc = (int)(rem / nc), ic = (int)(rem % nc);
  const size_t m = BRICK ? (size_t)oct_brick_index((unsigned)kc, (unsigned)jc, (unsigned)ic,
                                                   ((unsigned)nt + 2u) / 2u, (nc + 1u) / 2u)
                         : (size_t)kc * ks + (size_t)jc * js + ic;
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

template <bool BRICK>
__global__ void pack_gather_cart_kernel(const float* __restrict__ mu, int nz, int ny, int nx,
                                        unsigned ks, unsigned js, float4* __restrict__ oct, int kc0) {
  // cells (kc, jc, ic) in [0, n] per axis: corner (kc-1, jc-1, ic-1)
  const unsigned rem = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned nc = (unsigned)nx + 1u;
  if (rem >= (unsigned)(ny + 1) * nc) return;
  const int kc = kc0 + (int)blockIdx.y;
  const int jc = (int)(rem / nc), ic = (int)(rem % nc);
  const size_t m = BRICK ? (size_t)oct_brick_index((unsigned)kc, (unsigned)jc, (unsigned)ic,
                                                   ((unsigned)ny + 2u) / 2u, (nc + 1u) / 2u)
                         : (size_t)kc * ks + (size_t)jc * js + ic;
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

// GL_QUAD: cell (kc, jc, ic), kc in [0, nz+1]: the bilinear polynomial
// (c0, cr, ct, crt) of layer kc-1 (clamped; -1 and n are halo copies) over
// rows jc-1, jc (theta wraps / y clamps) and columns ic-1, ic (clamped).  The
// trilinear cell of layers k, k+1 is (L_k, L_k+1 - L_k): the same fp32 ops as
// trilinear_coeffs, so GL_QUAD, GL_OCT and the plain path agree bit for bit.
template <bool CYL>
__global__ void pack_vquad_kernel(const float* __restrict__ mu, int nk, int nj, int ni,
                                  unsigned ks, unsigned js, float4* __restrict__ q, int kc0) {
  const unsigned rem = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned nc = (unsigned)ni + 1u;
  if (rem >= (unsigned)(nj + 1) * nc) return;
  const int kc = kc0 + (int)blockIdx.y;
  const int jc = (int)(rem / nc), ic = (int)(rem % nc);
#if CT_QUAD_BRICK
  const size_t m = quad_brick_index((unsigned)kc, (unsigned)jc, (unsigned)ic,
                                    qbricks((unsigned)nj + 1u, QB_LJ), qbricks(nc, QB_LI));
#else
  const size_t m = (size_t)kc * ks + (size_t)jc * js + ic;
#endif
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

CellStrides gather_strides_cyl(const ct_cyl_grid& g) {
  return cell_strides((unsigned)CylGeo::gather_rows(g.n_theta), (unsigned)g.n_r + 1u);
}
CellStrides gather_strides_cart(const ct_cart_grid& g) {
  return cell_strides((unsigned)g.n_y + 1u, (unsigned)g.n_x + 1u);
}
double cells_layer_cyl(const ct_cyl_grid& g) {
  return (double)CylGeo::gather_rows(g.n_theta) * (g.n_r + 1);
}
double cells_layer_cart(const ct_cart_grid& g) { return (double)(g.n_y + 1) * (g.n_x + 1); }
// gather buffer length in floats: (n+1) layers x 8 floats, or GL_QUAD (n+2) x 4
// bricked GL_QUAD: ceil(layers/2) x ceil(rows/2) x ceil(cols/2) bricks of 8 cells
int64_t quad_brick_floats(int64_t layers, int64_t rows, int64_t cols) {
  return 32 * (int64_t)qbricks((unsigned)layers, QB_LK) * (int64_t)qbricks((unsigned)rows, QB_LJ) *
         (int64_t)qbricks((unsigned)cols, QB_LI);
}
int64_t gather_floats_cyl(const ct_cyl_grid& g) {
  if (CT_QUAD_BRICK && gather_quad(cells_layer_cyl(g)))
    return quad_brick_floats(g.n_h + 2, CylGeo::gather_rows(g.n_theta), g.n_r + 1);
  if (gather_obrick(cells_layer_cyl(g)))
    return 32 * (int64_t)(g.n_h + 1) * ((CylGeo::gather_rows(g.n_theta) + 1) / 2) *
           ((g.n_r + 2) / 2);
  const unsigned ks = gather_strides_cyl(g).ks;
  return gather_quad(cells_layer_cyl(g)) ? 4 * (int64_t)(g.n_h + 2) * ks
                                         : 8 * (int64_t)(g.n_h + 1) * ks;
}
int64_t gather_floats_cart(const ct_cart_grid& g) {
  if (CT_QUAD_BRICK && gather_quad(cells_layer_cart(g)))
    return quad_brick_floats(g.n_z + 2, g.n_y + 1, g.n_x + 1);
  if (gather_obrick(cells_layer_cart(g)))
    return 32 * (int64_t)(g.n_z + 1) * ((g.n_y + 2) / 2) * ((g.n_x + 2) / 2);
  const unsigned ks = gather_strides_cart(g).ks;
  return gather_quad(cells_layer_cart(g)) ? 4 * (int64_t)(g.n_z + 2) * ks
                                          : 8 * (int64_t)(g.n_z + 1) * ks;
}


// Residual partials at view-id slots (FpArgs::red_rows): the scratch of an
// identity-ordered batch of n_slots views, filled by launches over disjoint
// view sets / row ranges and summed once by ct_residual_sum.
int check_rows(const ct_batch* batch, int64_t row_lo, int64_t row_hi) {
  if (row_lo < 0 || row_hi <= row_lo || row_hi > (int64_t)batch->n_batch * batch->det_rows)
    return set_err(CT_ERR_ARG, "bad row range");
  return CT_OK;
}

int check_slots(const ct_batch* batch, int n_slots, const double* scratch) {
  if (!batch->view_ids) return set_err(CT_ERR_ARG, "residual slots need view ids");
  if (n_slots < 1 || n_slots > 65535) return set_err(CT_ERR_ARG, "bad residual slot count");
  if (!scratch) return set_err(CT_ERR_ARG, "null scratch");
  return CT_OK;
}

template <class Geo>
int fp_rows(const Geo& geo, const ct_ray_view* views, const ct_batch* batch,
            const ct_sampling* s, const float* p_meas, const double* row_thr, float* corr,
            int64_t row_lo, int64_t row_hi, int n_slots, double* scratch, ct_stream_t stream,
            float* const* peers = nullptr, int n_peers = 0, int64_t peer_off = 0) {
  int rc = check_rows(batch, row_lo, row_hi);
  if (rc) return rc;
  if (n_peers < 0 || (n_peers > 0 && !peers)) return set_err(CT_ERR_ARG, "bad peer list");
  if (corr && !scratch)
    return launch_fp<Geo, EPI_CORR>(geo, views, *batch, *s, p_meas, row_thr, corr, nullptr,
                                    nullptr, CT_STREAM(stream), 0, row_lo, row_hi, peers,
                                    n_peers, peer_off);
  if ((rc = check_slots(batch, n_slots, scratch))) return rc;
  if (corr)
    return launch_fp<Geo, EPI_CORR_RESID>(geo, views, *batch, *s, p_meas, row_thr, corr, nullptr,
                                          scratch, CT_STREAM(stream), n_slots, row_lo, row_hi,
                                          peers, n_peers, peer_off);
  return launch_fp<Geo, EPI_RESID>(geo, views, *batch, *s, p_meas, nullptr, nullptr, nullptr,
                                   scratch, CT_STREAM(stream), n_slots, row_lo, row_hi);
}

template <class Geo>
int launch_row_samples(const Geo& geo, const ct_ray_view* views, const ct_batch* batch,
                       const ct_sampling* s, uint64_t* out, ct_stream_t stream) {
  if (!out) return set_err(CT_ERR_ARG, "null row_samples");
  if (cudaMemsetAsync(out, 0, sizeof(uint64_t) * batch->n_batch * batch->det_rows,
                      CT_STREAM(stream)))
    return check_launch("memset");
  return launch_fp<Geo, EPI_ROWCOUNT>(geo, views, *batch, *s, nullptr, nullptr, nullptr, nullptr,
                                      reinterpret_cast<double*>(out), CT_STREAM(stream));
}

// Band launches (slab decomposition): corrections of view slot b's rows
// [bands[2b], bands[2b+1]) into the full [n][rows][cols] stack, with residual
// partials at the full launch's slots when a scratch is given.
template <class Geo>
int fp_bands(const Geo& geo, const ct_ray_view* views, const ct_batch* batch,
             const ct_sampling* s, const float* p_meas, const double* row_thr, float* corr,
             const int32_t* bands, int band_rows, int n_slots, double* scratch,
             ct_stream_t stream, float* const* peers = nullptr, int n_peers = 0,
             const int32_t* peer_rows = nullptr) {
  if (!bands) return set_err(CT_ERR_ARG, "null bands");
  if (band_rows < 1 || band_rows > batch->det_rows) return set_err(CT_ERR_ARG, "bad band_rows");
  if (n_peers < 0 || (n_peers > 0 && !peers)) return set_err(CT_ERR_ARG, "bad peer list");
  const cudaStream_t st = CT_STREAM(stream);
  if (corr && !scratch)
    return launch_fp<Geo, EPI_CORR>(geo, views, *batch, *s, p_meas, row_thr, corr, nullptr,
                                    nullptr, st, 0, 0, INT64_MAX, peers, n_peers, 0, bands,
                                    band_rows, peer_rows);
  int rc = check_slots(batch, n_slots, scratch);
  if (rc) return rc;
  if (corr)
    return launch_fp<Geo, EPI_CORR_RESID>(geo, views, *batch, *s, p_meas, row_thr, corr,
                                          nullptr, scratch, st, n_slots, 0, INT64_MAX, peers,
                                          n_peers, 0, bands, band_rows, peer_rows);
  return launch_fp<Geo, EPI_RESID>(geo, views, *batch, *s, p_meas, nullptr, nullptr, nullptr,
                                   scratch, st, n_slots, 0, INT64_MAX, nullptr, 0, 0, bands,
                                   band_rows);
}

// FP cell layers of a ray: the layer index kc = floor(fh1) of the gather
// cell every sample reads (the march's own fp32 h index, CylGeo::locate /
// CartGeo::locate); monotone in the sample index, so the ray's extremes are
// its first and last samples.
__device__ __forceinline__ int cell_layer_of(const CylGeo&, const RayF& ry, float k) {
  return (int)(__float_as_uint(__fadd_rd(fmaf(k, ry.ih, ry.eh), 8388608.0f)) - kMagicBits);
}
__device__ __forceinline__ int cell_layer_of(const CartGeo& g, const RayF& ry, float k) {
  const float fz1 = fmaf(fmaf(k, ry.iz, ry.ez), g.inv_vs, g.off1[2]);
  return (int)(__float_as_uint(__fadd_rd(fz1, 8388608.0f)) - kMagicBits);
}

// per (view slot, detector row): [min, max] FP cell layer over the row's rays
// and sub-rays (rows without samples keep INT_MAX / INT_MIN)
template <class Geo>
__global__ void row_cells_kernel(const Geo geo, const ct_ray_view* __restrict__ views,
                                 const int32_t* __restrict__ view_ids, int rows, int cols,
                                 int ss, double step, int* __restrict__ out) {
  const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  int lo = INT_MAX, hi = INT_MIN;
  int row = 0;
  if (pix < (int64_t)rows * cols) {
    row = (int)(pix / cols);
    const int col = (int)(pix % cols);
    const ct_ray_view& v = views[view_ids ? view_ids[b] : b];
    for (int sv = 0; sv < ss; ++sv) {
      const double off_v = ss == 1 ? 0.0 : dsub(ddiv((double)sv + 0.5, (double)ss), 0.5);
      for (int su = 0; su < ss; ++su) {
        const double off_u = ss == 1 ? 0.0 : dsub(ddiv((double)su + 0.5, (double)ss), 0.5);
        double d[3], t0, t1;
        subray_dir(v, dadd((double)col, off_u), dadd((double)row, off_v), d);
        if (!geo.interval(v.src, d, t0, t1) || !(t1 > t0)) continue;
        const int n = (int)ceil(ddiv(dsub(t1, t0), step));
        const double ts = dadd(t0, dmul(0.5, step));
        double e[3], inc[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          e[a] = v.src[a] + ts * d[a];
          inc[a] = step * d[a];
        }
        RayF ry;
        geo.setup_ray(e, inc, n, ry);
        const int k0 = cell_layer_of(geo, ry, 0.0f), k1 = cell_layer_of(geo, ry, (float)(n - 1));
        lo = min(lo, min(k0, k1));
        hi = max(hi, max(k0, k1));
      }
    }
  }
  if (lo <= hi) {
    atomicMin(out + 2 * ((int64_t)b * rows + row), lo);
    atomicMax(out + 2 * ((int64_t)b * rows + row) + 1, hi);
  }
}

__global__ void fill_cells_kernel(int* out, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = (i & 1) ? INT_MIN : INT_MAX;
}

template <class Geo>
int launch_row_cells(const Geo& geo, const ct_ray_view* views, const ct_batch* batch,
                     const ct_sampling* s, int32_t* out, ct_stream_t stream) {
  if (!out) return set_err(CT_ERR_ARG, "null row cells");
  const cudaStream_t st = CT_STREAM(stream);
  const int64_t n = 2LL * batch->n_batch * batch->det_rows;
  fill_cells_kernel<<<blocks_for(n, 256), 256, 0, st>>>(out, n);
  const int64_t npix = (int64_t)batch->det_rows * batch->det_cols;
  row_cells_kernel<Geo><<<dim3(blocks_for(npix, 256), batch->n_batch), 256, 0, st>>>(
      geo, views, batch->view_ids, batch->det_rows, batch->det_cols, s->supersample, s->step,
      out);
  return check_launch("row_cells_kernel");
}

}  // namespace

extern "C" {

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

int ct_fp_row_tile(const ct_batch* batch) {
  if (!batch || batch->det_rows < 1 || batch->det_cols < 1) return 0;
  return FP_WY * tile_wh(lanes_for(batch->det_rows, batch->det_cols));
}

int ct_fp_cyl_correction_rows(const float* mu, const float* gather, const ct_cyl_grid* grid,
                              const ct_ray_view* views, const ct_batch* batch,
                              const ct_sampling* s, const float* p_meas, const double* row_thr,
                              float* corr, int64_t row_lo, int64_t row_hi, int n_slots,
                              double* scratch, float* const* corr_peers, int n_peers,
                              int64_t peer_offset, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cyl(grid))) return rc;
  if (!mu || !p_meas || !row_thr || !corr) return set_err(CT_ERR_ARG, "null pointer");
  CylGeo geo;
  geo.init(mu, gather, *grid);
  return fp_rows(geo, views, batch, s, p_meas, row_thr, corr, row_lo, row_hi, n_slots, scratch,
                 stream, corr_peers, n_peers, peer_offset);
}

int ct_fp_cart_correction_rows(const float* mu, const float* gather, const ct_cart_grid* grid,
                               const ct_ray_view* views, const ct_batch* batch,
                               const ct_sampling* s, const float* p_meas, const double* row_thr,
                               float* corr, int64_t row_lo, int64_t row_hi, int n_slots,
                               double* scratch, float* const* corr_peers, int n_peers,
                              int64_t peer_offset, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cart(grid))) return rc;
  if (!mu || !p_meas || !row_thr || !corr) return set_err(CT_ERR_ARG, "null pointer");
  CartGeo geo;
  geo.init(mu, gather, *grid);
  return fp_rows(geo, views, batch, s, p_meas, row_thr, corr, row_lo, row_hi, n_slots, scratch,
                 stream, corr_peers, n_peers, peer_offset);
}

int ct_fp_cyl_residual_rows(const float* mu, const float* gather, const ct_cyl_grid* grid,
                            const ct_ray_view* views, const ct_batch* batch,
                            const ct_sampling* s, const float* p_meas, int64_t row_lo,
                            int64_t row_hi, int n_slots, double* scratch, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cyl(grid))) return rc;
  if (!mu || !p_meas || !scratch) return set_err(CT_ERR_ARG, "null pointer");
  CylGeo geo;
  geo.init(mu, gather, *grid);
  return fp_rows(geo, views, batch, s, p_meas, nullptr, nullptr, row_lo, row_hi, n_slots,
                 scratch, stream);
}

int ct_fp_cart_residual_rows(const float* mu, const float* gather, const ct_cart_grid* grid,
                             const ct_ray_view* views, const ct_batch* batch,
                             const ct_sampling* s, const float* p_meas, int64_t row_lo,
                             int64_t row_hi, int n_slots, double* scratch, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cart(grid))) return rc;
  if (!mu || !p_meas || !scratch) return set_err(CT_ERR_ARG, "null pointer");
  CartGeo geo;
  geo.init(mu, gather, *grid);
  return fp_rows(geo, views, batch, s, p_meas, nullptr, nullptr, row_lo, row_hi, n_slots,
                 scratch, stream);
}

int ct_residual_sum(const double* scratch, int64_t n, double* accum, ct_stream_t stream) {
  if (!scratch || !accum || n < 1) return set_err(CT_ERR_ARG, "bad residual sum arguments");
  sum_partials_kernel<<<1, 1024, 0, CT_STREAM(stream)>>>(scratch, n, accum);
  return check_launch("sum_partials_kernel");
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

int ct_fp_cyl_correction_bands(const float* mu, const float* gather, const ct_cyl_grid* grid,
                               const ct_ray_view* views, const ct_batch* batch,
                               const ct_sampling* s, const float* p_meas, const double* row_thr,
                               float* corr, const int32_t* bands, int band_rows, int n_slots,
                               double* scratch, float* const* corr_peers,
    int n_peers, const int32_t* peer_rows, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cyl(grid))) return rc;
  if (!mu || !p_meas || !row_thr || !corr) return set_err(CT_ERR_ARG, "null pointer");
  CylGeo geo;
  geo.init(mu, gather, *grid);
  return fp_bands(geo, views, batch, s, p_meas, row_thr, corr, bands, band_rows, n_slots,
                  scratch, stream, corr_peers, n_peers, peer_rows);
}

int ct_fp_cart_correction_bands(const float* mu, const float* gather, const ct_cart_grid* grid,
                                const ct_ray_view* views, const ct_batch* batch,
                                const ct_sampling* s, const float* p_meas, const double* row_thr,
                                float* corr, const int32_t* bands, int band_rows, int n_slots,
                                double* scratch, float* const* corr_peers,
    int n_peers, const int32_t* peer_rows, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cart(grid))) return rc;
  if (!mu || !p_meas || !row_thr || !corr) return set_err(CT_ERR_ARG, "null pointer");
  CartGeo geo;
  geo.init(mu, gather, *grid);
  return fp_bands(geo, views, batch, s, p_meas, row_thr, corr, bands, band_rows, n_slots,
                  scratch, stream, corr_peers, n_peers, peer_rows);
}

int ct_fp_cyl_residual_bands(const float* mu, const float* gather, const ct_cyl_grid* grid,
                             const ct_ray_view* views, const ct_batch* batch,
                             const ct_sampling* s, const float* p_meas, const int32_t* bands,
                             int band_rows, int n_slots, double* scratch, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cyl(grid))) return rc;
  if (!mu || !p_meas || !scratch) return set_err(CT_ERR_ARG, "null pointer");
  CylGeo geo;
  geo.init(mu, gather, *grid);
  return fp_bands(geo, views, batch, s, p_meas, nullptr, nullptr, bands, band_rows, n_slots,
                  scratch, stream);
}

int ct_fp_cart_residual_bands(const float* mu, const float* gather, const ct_cart_grid* grid,
                              const ct_ray_view* views, const ct_batch* batch,
                              const ct_sampling* s, const float* p_meas, const int32_t* bands,
                              int band_rows, int n_slots, double* scratch, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cart(grid))) return rc;
  if (!mu || !p_meas || !scratch) return set_err(CT_ERR_ARG, "null pointer");
  CartGeo geo;
  geo.init(mu, gather, *grid);
  return fp_bands(geo, views, batch, s, p_meas, nullptr, nullptr, bands, band_rows, n_slots,
                  scratch, stream);
}

int ct_row_cells_cyl(const ct_cyl_grid* grid, const ct_ray_view* views, const ct_batch* batch,
                     const ct_sampling* s, int32_t* cells, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cyl(grid))) return rc;
  CylGeo geo;
  geo.init(nullptr, nullptr, *grid);
  return launch_row_cells(geo, views, batch, s, cells, stream);
}

int ct_row_cells_cart(const ct_cart_grid* grid, const ct_ray_view* views, const ct_batch* batch,
                      const ct_sampling* s, int32_t* cells, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cart(grid))) return rc;
  CartGeo geo;
  geo.init(nullptr, nullptr, *grid);
  return launch_row_cells(geo, views, batch, s, cells, stream);
}

int ct_row_samples_cyl(const ct_cyl_grid* grid, const ct_ray_view* views, const ct_batch* batch,
                       const ct_sampling* s, uint64_t* row_samples, ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cyl(grid))) return rc;
  CylGeo geo;
  geo.init(nullptr, nullptr, *grid);
  return launch_row_samples(geo, views, batch, s, row_samples, stream);
}

int ct_row_samples_cart(const ct_cart_grid* grid, const ct_ray_view* views,
                        const ct_batch* batch, const ct_sampling* s, uint64_t* row_samples,
                        ct_stream_t stream) {
  int rc = check_batch(batch, views, s);
  if (rc || (rc = check_cart(grid))) return rc;
  CartGeo geo;
  geo.init(nullptr, nullptr, *grid);
  return launch_row_samples(geo, views, batch, s, row_samples, stream);
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

int64_t ct_gather_floats_cyl(const ct_cyl_grid* grid) {
  return check_cyl(grid) ? 0 : gather_floats_cyl(*grid);
}

int64_t ct_gather_floats_cart(const ct_cart_grid* grid) {
  return check_cart(grid) ? 0 : gather_floats_cart(*grid);
}

static int layout_of(double cells) {
  return gather_quad(cells) ? CT_GL_QUAD : gather_obrick(cells) ? CT_GL_OCTB : CT_GL_OCT;
}
static_assert(CT_GL_OCT == GL_OCT && CT_GL_QUAD == GL_QUAD && CT_GL_OCTB == GL_OCTB,
              "layout enum");

int ct_gather_layout_cyl(const ct_cyl_grid* grid) {
  return check_cyl(grid) ? CT_ERR_ARG : layout_of(cells_layer_cyl(*grid));
}

int ct_gather_layout_cart(const ct_cart_grid* grid) {
  return check_cart(grid) ? CT_ERR_ARG : layout_of(cells_layer_cart(*grid));
}

static int pack_cyl_layers(const float* mu, const ct_cyl_grid* grid, float* gather,
                             int kc_lo, int kc_hi,
                       ct_stream_t stream) {
  int rc = check_cyl(grid);
  if (rc) return rc;
  if (!mu || !gather) return set_err(CT_ERR_ARG, "null mu/gather");
  if (reinterpret_cast<uintptr_t>(gather) % 16) return set_err(CT_ERR_ARG, "gather not 16B-aligned");
  if (grid->n_h + 2 > 65535) return set_err(CT_ERR_ARG, "gather layout: n_h + 2 > 65535");
  const CellStrides cs = gather_strides_cyl(*grid);
  const double cells = cells_layer_cyl(*grid);
  if (CT_QUAD_BRICK && gather_quad(cells) &&
      quad_brick_floats(grid->n_h + 2, grid->n_theta + 1, grid->n_r + 1) / 4 >= 2147483648LL)
    return set_err(CT_ERR_ARG, "gather layout too large for 32-bit brick indices");
  const unsigned nb = blocks_for((int64_t)cells, 256);
  // FP cell layers [kc_lo, kc_hi]: GL_QUAD cells read quad layers kc, kc + 1
  const bool q = gather_quad(cells);
  const int k0 = max(kc_lo, 0), k1 = min(q ? kc_hi + 1 : kc_hi, grid->n_h + (q ? 1 : 0));
  if (k1 < k0) return CT_OK;
  const unsigned nl = (unsigned)(k1 - k0 + 1);
  if (q) {
    pack_vquad_kernel<true><<<dim3(nb, nl), 256, 0, CT_STREAM(stream)>>>(
        mu, grid->n_h, grid->n_theta, grid->n_r, cs.ks, cs.js, reinterpret_cast<float4*>(gather), k0);
    return check_launch("pack_vquad_kernel");
  }
  if (gather_obrick(cells))
    pack_gather_cyl_kernel<true><<<dim3(nb, nl), 256, 0, CT_STREAM(stream)>>>(
        mu, grid->n_h, grid->n_theta, grid->n_r, cs.ks, cs.js, reinterpret_cast<float4*>(gather), k0);
  else
    pack_gather_cyl_kernel<false><<<dim3(nb, nl), 256, 0, CT_STREAM(stream)>>>(
        mu, grid->n_h, grid->n_theta, grid->n_r, cs.ks, cs.js, reinterpret_cast<float4*>(gather), k0);
  return check_launch("pack_gather_cyl_kernel");
}

int ct_pack_gather_cyl(const float* mu, const ct_cyl_grid* grid, float* gather,
                        ct_stream_t stream) {
  if (!grid) return set_err(CT_ERR_ARG, "null grid");
  return pack_cyl_layers(mu, grid, gather, 0, grid->n_h, stream);
}

int ct_pack_gather_cyl_layers(const float* mu, const ct_cyl_grid* grid, float* gather,
                               int32_t kc_lo, int32_t kc_hi, ct_stream_t stream) {
  if (!grid) return set_err(CT_ERR_ARG, "null grid");
  return pack_cyl_layers(mu, grid, gather, kc_lo, kc_hi, stream);
}

static int pack_cart_layers(const float* mu, const ct_cart_grid* grid, float* gather,
                             int kc_lo, int kc_hi,
                        ct_stream_t stream) {
  int rc = check_cart(grid);
  if (rc) return rc;
  if (!mu || !gather) return set_err(CT_ERR_ARG, "null mu/gather");
  if (reinterpret_cast<uintptr_t>(gather) % 16) return set_err(CT_ERR_ARG, "gather not 16B-aligned");
  if (grid->n_z + 2 > 65535) return set_err(CT_ERR_ARG, "gather layout: n_z + 2 > 65535");
  const CellStrides cs = gather_strides_cart(*grid);
  const double cells = cells_layer_cart(*grid);
  if (CT_QUAD_BRICK && gather_quad(cells) &&
      quad_brick_floats(grid->n_z + 2, grid->n_y + 1, grid->n_x + 1) / 4 >= 2147483648LL)
    return set_err(CT_ERR_ARG, "gather layout too large for 32-bit brick indices");
  const unsigned nb = blocks_for((int64_t)cells, 256);
  // FP cell layers [kc_lo, kc_hi]: GL_QUAD cells read quad layers kc, kc + 1
  const bool q = gather_quad(cells);
  const int k0 = max(kc_lo, 0), k1 = min(q ? kc_hi + 1 : kc_hi, grid->n_z + (q ? 1 : 0));
  if (k1 < k0) return CT_OK;
  const unsigned nl = (unsigned)(k1 - k0 + 1);
  if (q) {
    pack_vquad_kernel<false><<<dim3(nb, nl), 256, 0, CT_STREAM(stream)>>>(
        mu, grid->n_z, grid->n_y, grid->n_x, cs.ks, cs.js, reinterpret_cast<float4*>(gather), k0);
    return check_launch("pack_vquad_kernel");
  }
  if (gather_obrick(cells))
    pack_gather_cart_kernel<true><<<dim3(nb, nl), 256, 0, CT_STREAM(stream)>>>(
        mu, grid->n_z, grid->n_y, grid->n_x, cs.ks, cs.js, reinterpret_cast<float4*>(gather), k0);
  else
    pack_gather_cart_kernel<false><<<dim3(nb, nl), 256, 0, CT_STREAM(stream)>>>(
        mu, grid->n_z, grid->n_y, grid->n_x, cs.ks, cs.js, reinterpret_cast<float4*>(gather), k0);
  return check_launch("pack_gather_cart_kernel");
}

int ct_pack_gather_cart(const float* mu, const ct_cart_grid* grid, float* gather,
                        ct_stream_t stream) {
  if (!grid) return set_err(CT_ERR_ARG, "null grid");
  return pack_cart_layers(mu, grid, gather, 0, grid->n_z, stream);
}

int ct_pack_gather_cart_layers(const float* mu, const ct_cart_grid* grid, float* gather,
                               int32_t kc_lo, int32_t kc_hi, ct_stream_t stream) {
  if (!grid) return set_err(CT_ERR_ARG, "null grid");
  return pack_cart_layers(mu, grid, gather, kc_lo, kc_hi, stream);
}

}  // extern "C"
