// ct_pose.cu -- projection-image statistics of the pose step (imgproc.py,
// posefit.py).
#include "ct_common.cuh"

namespace {

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


}  // namespace

extern "C" {

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
