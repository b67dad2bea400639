// ct_sample.cu -- point sampling / resampling (grid.py:261-319) and the
// Beer-Lambert conversion (projector.py:169-181).
#include "ct_common.cuh"

namespace {

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



}  // namespace

extern "C" {

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

}  // extern "C"
