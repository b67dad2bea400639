/*
 * cyltomo_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, float64 restatement of the reference's numba kernels
 * (/root/reference/pkg/src/cyltomo/_kernels.py).  It is the CPU checker for
 * the B200 kernels: only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load it.  The product path never
 * links or calls it.
 *
 * Parity is PINNED: tests/test_oracle_golden.py compares every entry point
 * below against golden vectors produced by running the unmodified reference
 * (tests/golden/make_golden.py), to 0 ulp on the FP sample counts and
 * <=1e-12 relative on values.
 *
 * Build: see oracle/Makefile (gcc -O2 -fopenmp -ffp-contract=off), so that
 * a*b+c is never fused -- the reference (numba, fastmath off) does not fuse
 * either, which keeps the per-ray interval arithmetic bit-identical.
 *
 * Conventions (reference cyltomo/_kernels.py:11-14): cylindrical volumes are
 * mu[h][theta][r] (r fastest), cell centres at h=(k+.5)dh-H/2,
 * theta=(j+.5)dtheta, r=(m+.5)dr.  Cartesian volumes are mu[z][y][x] with
 * centres origin+(i+.5)*voxel.
 */
#include <math.h>
#include <stdint.h>
#include <stddef.h>

#define OR_TWO_PI (2.0 * 3.14159265358979323846)

/* Python's floor-modulo for ints (result carries the divisor's sign). */
static inline int64_t pymod(int64_t a, int64_t n) {
    int64_t m = a % n;
    return m < 0 ? m + n : m;
}

/* _kernels.py:35-45 -- snap an index within 1e-9 of an integer onto it.
 * Python's round() is round-half-even == rint() in the default FP mode. */
static inline double snap_index(double f) {
    double r = rint(f);
    return fabs(f - r) < 1e-9 ? r : f;
}

static inline double clampd(double f, double lo, double hi) {
    if (f < lo) return lo;
    if (f > hi) return hi;
    return f;
}

/* _kernels.py:48-107 -- trilinear sample of a cylindrical volume at grid
 * coordinates (r, theta, h); theta wraps, r/h clamp, outside support -> 0. */
double oracle_interp_cyl(const double *mu, int64_t nh, int64_t nt, int64_t nr,
                         double radius, double height,
                         double r, double th, double h, int nearest) {
    const double half_h = 0.5 * height;
    if (r > radius || h < -half_h || h > half_h) return 0.0;
    const double dr = radius / (double)nr;
    const double dth = OR_TWO_PI / (double)nt;
    const double dh = height / (double)nh;
    double fr = clampd(snap_index(r / dr - 0.5), 0.0, (double)nr - 1.0);
    double fh = clampd(snap_index((h + half_h) / dh - 0.5), 0.0, (double)nh - 1.0);
    double ft = snap_index(th / dth - 0.5);
    if (nearest) {
        int64_t ir = (int64_t)rint(fr);
        int64_t ih = (int64_t)rint(fh);
        int64_t it = pymod((int64_t)rint(ft), nt);
        return mu[(ih * nt + it) * nr + ir];
    }
    int64_t i0 = (int64_t)floor(fr);
    double wr = fr - (double)i0;
    int64_t i1 = i0 + 1 > nr - 1 ? nr - 1 : i0 + 1;
    int64_t k0 = (int64_t)floor(fh);
    double wh = fh - (double)k0;
    int64_t k1 = k0 + 1 > nh - 1 ? nh - 1 : k0 + 1;
    int64_t jf = (int64_t)floor(ft);
    double wt = ft - (double)jf;
    int64_t j0 = pymod(jf, nt);
    int64_t j1 = j0 + 1 == nt ? 0 : j0 + 1;
#define MU(k, j, i) mu[((k) * nt + (j)) * nr + (i)]
    double c00 = MU(k0, j0, i0) * (1.0 - wr) + MU(k0, j0, i1) * wr;
    double c01 = MU(k0, j1, i0) * (1.0 - wr) + MU(k0, j1, i1) * wr;
    double c10 = MU(k1, j0, i0) * (1.0 - wr) + MU(k1, j0, i1) * wr;
    double c11 = MU(k1, j1, i0) * (1.0 - wr) + MU(k1, j1, i1) * wr;
#undef MU
    double c0 = c00 * (1.0 - wt) + c01 * wt;
    double c1 = c10 * (1.0 - wt) + c11 * wt;
    return c0 * (1.0 - wh) + c1 * wh;
}

/* _kernels.py:110-151 -- trilinear sample of a Cartesian volume (world). */
double oracle_interp_cart(const double *mu, int64_t nz, int64_t ny, int64_t nx,
                          double vs, double ox, double oy, double oz,
                          double x, double y, double z, int nearest) {
    double fx = snap_index((x - ox) / vs - 0.5);
    double fy = snap_index((y - oy) / vs - 0.5);
    double fz = snap_index((z - oz) / vs - 0.5);
    if (fx < -0.5 || fx > (double)nx - 0.5 || fy < -0.5 || fy > (double)ny - 0.5 ||
        fz < -0.5 || fz > (double)nz - 0.5)
        return 0.0;
    fx = clampd(fx, 0.0, (double)nx - 1.0);
    fy = clampd(fy, 0.0, (double)ny - 1.0);
    fz = clampd(fz, 0.0, (double)nz - 1.0);
    if (nearest)
        return mu[((int64_t)rint(fz) * ny + (int64_t)rint(fy)) * nx + (int64_t)rint(fx)];
    int64_t i0 = (int64_t)floor(fx), j0 = (int64_t)floor(fy), k0 = (int64_t)floor(fz);
    double wx = fx - (double)i0, wy = fy - (double)j0, wz = fz - (double)k0;
    int64_t i1 = i0 + 1 < nx - 1 ? i0 + 1 : nx - 1;
    int64_t j1 = j0 + 1 < ny - 1 ? j0 + 1 : ny - 1;
    int64_t k1 = k0 + 1 < nz - 1 ? k0 + 1 : nz - 1;
#define MU(k, j, i) mu[((k) * ny + (j)) * nx + (i)]
    double c00 = MU(k0, j0, i0) * (1.0 - wx) + MU(k0, j0, i1) * wx;
    double c01 = MU(k0, j1, i0) * (1.0 - wx) + MU(k0, j1, i1) * wx;
    double c10 = MU(k1, j0, i0) * (1.0 - wx) + MU(k1, j0, i1) * wx;
    double c11 = MU(k1, j1, i0) * (1.0 - wx) + MU(k1, j1, i1) * wx;
#undef MU
    double c0 = c00 * (1.0 - wy) + c01 * wy;
    double c1 = c10 * (1.0 - wy) + c11 * wy;
    return c0 * (1.0 - wz) + c1 * wz;
}

/* _kernels.py:154-163 */
void oracle_sample_cyl_many(const double *mu, int64_t nh, int64_t nt, int64_t nr,
                            double radius, double height, const double *rs,
                            const double *ths, const double *hs, int64_t n,
                            int nearest, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        out[i] = oracle_interp_cyl(mu, nh, nt, nr, radius, height, rs[i], ths[i], hs[i], nearest);
}

void oracle_sample_cart_many(const double *mu, int64_t nz, int64_t ny, int64_t nx,
                             double vs, double ox, double oy, double oz,
                             const double *xs, const double *ys, const double *zs,
                             int64_t n, int nearest, double *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i)
        out[i] = oracle_interp_cart(mu, nz, ny, nx, vs, ox, oy, oz, xs[i], ys[i], zs[i], nearest);
}

/* _kernels.py:170-204 -- ray vs finite cylinder, t clamped >= 0. */
static void cylinder_interval(double sx, double sy, double sz, double dx, double dy,
                              double dz, double radius, double half_h,
                              double *t0_out, double *t1_out) {
    double tr0, tr1, tz0, tz1;
    double a = dx * dx + dy * dy;
    if (a < 1e-18) {
        if (sx * sx + sy * sy > radius * radius) { *t0_out = 0.0; *t1_out = -1.0; return; }
        tr0 = -1e30; tr1 = 1e30;
    } else {
        double b = sx * dx + sy * dy;
        double c = sx * sx + sy * sy - radius * radius;
        double disc = b * b - a * c;
        if (disc <= 0.0) { *t0_out = 0.0; *t1_out = -1.0; return; }
        double sq = sqrt(disc);
        tr0 = (-b - sq) / a;
        tr1 = (-b + sq) / a;
    }
    if (fabs(dz) < 1e-18) {
        if (fabs(sz) > half_h) { *t0_out = 0.0; *t1_out = -1.0; return; }
        tz0 = -1e30; tz1 = 1e30;
    } else {
        tz0 = (-half_h - sz) / dz;
        tz1 = (half_h - sz) / dz;
        if (tz0 > tz1) { double tmp = tz0; tz0 = tz1; tz1 = tmp; }
    }
    double t0 = tr0 > tz0 ? tr0 : tz0;
    if (t0 < 0.0) t0 = 0.0;
    *t0_out = t0;
    *t1_out = tr1 < tz1 ? tr1 : tz1;
}

/* _kernels.py:207-231 -- slab test against an axis-aligned box. */
static void box_interval(const double s[3], const double d[3], const double lo[3],
                         const double hi[3], double *t0_out, double *t1_out) {
    double t0 = 0.0, t1 = 1e30;
    for (int ax = 0; ax < 3; ++ax) {
        if (fabs(d[ax]) < 1e-18) {
            if (s[ax] < lo[ax] || s[ax] > hi[ax]) { *t0_out = 0.0; *t1_out = -1.0; return; }
        } else {
            double ta = (lo[ax] - s[ax]) / d[ax];
            double tb = (hi[ax] - s[ax]) / d[ax];
            if (ta > tb) { double tmp = ta; ta = tb; tb = tmp; }
            if (ta > t0) t0 = ta;
            if (tb < t1) t1 = tb;
        }
    }
    *t0_out = t0;
    *t1_out = t1;
}

/* Unit direction of the sub-ray through detector point (cu, cv)
 * (_kernels.py:263-272). */
static inline void subray_dir(const double src[3], const double org[3], const double du[3],
                              const double dv[3], double cu, double cv, double d[3]) {
    double px = org[0] + cu * du[0] + cv * dv[0];
    double py = org[1] + cu * du[1] + cv * dv[1];
    double pz = org[2] + cu * du[2] + cv * dv[2];
    double dx = px - src[0], dy = py - src[1], dz = pz - src[2];
    double norm = sqrt(dx * dx + dy * dy + dz * dz);
    d[0] = dx / norm; d[1] = dy / norm; d[2] = dz / norm;
}

/* One detector pixel of forward_cyl (_kernels.py:250-293).  Returns the
 * raw sums; *count gets the in-support sample count over all sub-rays. */
static void fp_cyl_pixel(const double *mu, int64_t nh, int64_t nt, int64_t nr,
                         double radius, double height, const double src[3],
                         const double org[3], const double du[3], const double dv[3],
                         int64_t row, int64_t col, double step, int ss, int nearest,
                         double *p, double *w) {
    const double half_h = 0.5 * height;
    const double inv_ss2 = 1.0 / (double)(ss * ss);
    double acc = 0.0, wacc = 0.0;
    for (int sv = 0; sv < ss; ++sv) {
        double off_v = ((double)sv + 0.5) / (double)ss - 0.5;
        for (int su = 0; su < ss; ++su) {
            double off_u = ((double)su + 0.5) / (double)ss - 0.5;
            double d[3];
            subray_dir(src, org, du, dv, (double)col + off_u, (double)row + off_v, d);
            double t0, t1;
            cylinder_interval(src[0], src[1], src[2], d[0], d[1], d[2], radius, half_h, &t0, &t1);
            if (t1 <= t0) continue;
            int64_t n = (int64_t)ceil((t1 - t0) / step);
            for (int64_t k = 0; k < n; ++k) {
                double t = t0 + ((double)k + 0.5) * step;
                double x = src[0] + t * d[0];
                double y = src[1] + t * d[1];
                double z = src[2] + t * d[2];
                double r = sqrt(x * x + y * y);
                if (r > radius || z < -half_h || z > half_h) continue;
                double th = atan2(y, x);
                if (th < 0.0) th += OR_TWO_PI;
                acc += oracle_interp_cyl(mu, nh, nt, nr, radius, height, r, th, z, nearest);
                wacc += 1.0;
            }
        }
    }
    *p = acc * step * inv_ss2;
    *w = wacc * step * inv_ss2;
}

/* _kernels.py:238-293 -- pixel-driven FP, grid-aligned frame, overwrites. */
void oracle_forward_cyl(const double *mu, int64_t nh, int64_t nt, int64_t nr,
                        double radius, double height, const double *a_src,
                        const double *a_origin, const double *a_du, const double *a_dv,
                        int64_t n_rows, int64_t n_cols, double step, int ss, int nearest,
                        double *out_p, double *out_w) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t pix = 0; pix < n_rows * n_cols; ++pix)
        fp_cyl_pixel(mu, nh, nt, nr, radius, height, a_src, a_origin, a_du, a_dv,
                     pix / n_cols, pix % n_cols, step, ss, nearest, &out_p[pix], &out_w[pix]);
}

/* The same per-pixel function on an explicit pixel list (for sampled parity
 * at sizes where a whole view is too slow on the CPU). */
void oracle_forward_cyl_pixels(const double *mu, int64_t nh, int64_t nt, int64_t nr,
                               double radius, double height, const double *a_src,
                               const double *a_origin, const double *a_du,
                               const double *a_dv, const int64_t *rows,
                               const int64_t *cols, int64_t n_pix, double step, int ss,
                               int nearest, double *out_p, double *out_w) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < n_pix; ++i)
        fp_cyl_pixel(mu, nh, nt, nr, radius, height, a_src, a_origin, a_du, a_dv,
                     rows[i], cols[i], step, ss, nearest, &out_p[i], &out_w[i]);
}

/* One pixel of forward_cart (_kernels.py:296-343). */
static void fp_cart_pixel(const double *mu, int64_t nz, int64_t ny, int64_t nx,
                          double vs, double ox, double oy, double oz, const double src[3],
                          const double org[3], const double du[3], const double dv[3],
                          int64_t row, int64_t col, double step, int ss, int nearest,
                          double *p, double *w) {
    const double lo[3] = {ox, oy, oz};
    const double hi[3] = {ox + (double)nx * vs, oy + (double)ny * vs, oz + (double)nz * vs};
    const double inv_ss2 = 1.0 / (double)(ss * ss);
    double acc = 0.0, wacc = 0.0;
    for (int sv = 0; sv < ss; ++sv) {
        double off_v = ((double)sv + 0.5) / (double)ss - 0.5;
        for (int su = 0; su < ss; ++su) {
            double off_u = ((double)su + 0.5) / (double)ss - 0.5;
            double d[3];
            subray_dir(src, org, du, dv, (double)col + off_u, (double)row + off_v, d);
            double t0, t1;
            box_interval(src, d, lo, hi, &t0, &t1);
            if (t1 <= t0) continue;
            int64_t n = (int64_t)ceil((t1 - t0) / step);
            for (int64_t k = 0; k < n; ++k) {
                double t = t0 + ((double)k + 0.5) * step;
                double x = src[0] + t * d[0];
                double y = src[1] + t * d[1];
                double z = src[2] + t * d[2];
                if (x < lo[0] || x > hi[0] || y < lo[1] || y > hi[1] || z < lo[2] || z > hi[2])
                    continue;
                acc += oracle_interp_cart(mu, nz, ny, nx, vs, ox, oy, oz, x, y, z, nearest);
                wacc += 1.0;
            }
        }
    }
    *p = acc * step * inv_ss2;
    *w = wacc * step * inv_ss2;
}

void oracle_forward_cart(const double *mu, int64_t nz, int64_t ny, int64_t nx, double vs,
                         double ox, double oy, double oz, const double *src,
                         const double *origin, const double *du, const double *dv,
                         int64_t n_rows, int64_t n_cols, double step, int ss, int nearest,
                         double *out_p, double *out_w) {
#pragma omp parallel for schedule(dynamic, 64)
    for (int64_t pix = 0; pix < n_rows * n_cols; ++pix)
        fp_cart_pixel(mu, nz, ny, nx, vs, ox, oy, oz, src, origin, du, dv, pix / n_cols,
                      pix % n_cols, step, ss, nearest, &out_p[pix], &out_w[pix]);
}

void oracle_forward_cart_pixels(const double *mu, int64_t nz, int64_t ny, int64_t nx,
                                double vs, double ox, double oy, double oz,
                                const double *src, const double *origin, const double *du,
                                const double *dv, const int64_t *rows, const int64_t *cols,
                                int64_t n_pix, double step, int ss, int nearest,
                                double *out_p, double *out_w) {
#pragma omp parallel for schedule(dynamic, 16)
    for (int64_t i = 0; i < n_pix; ++i)
        fp_cart_pixel(mu, nz, ny, nx, vs, ox, oy, oz, src, origin, du, dv, rows[i], cols[i],
                      step, ss, nearest, &out_p[i], &out_w[i]);
}

/* _kernels.py:350-377 -- bilinear footprint over in-bounds taps only. */
static inline void bilinear_gather(const double *img, int64_t n_rows, int64_t n_cols,
                                   double u, double v, double *num, double *den) {
    int64_t iu = (int64_t)floor(u);
    int64_t iv = (int64_t)floor(v);
    double fu = u - (double)iu, fv = v - (double)iv;
    double a = 0.0, b = 0.0;
    for (int dvv = 0; dvv < 2; ++dvv) {
        int64_t rr = iv + dvv;
        if (rr < 0 || rr >= n_rows) continue;
        double wv = dvv == 1 ? fv : 1.0 - fv;
        for (int duu = 0; duu < 2; ++duu) {
            int64_t cc = iu + duu;
            if (cc < 0 || cc >= n_cols) continue;
            double wu = duu == 1 ? fu : 1.0 - fu;
            double w = wu * wv;
            a += w * img[rr * n_cols + cc];
            b += w;
        }
    }
    *num = a;
    *den = b;
}

/* _kernels.py:380-417 -- voxel-driven BP of voxel m (one body of the prange
 * loop); adds its footprint to *num / *den. */
static inline void bp_cyl_voxel(int64_t m, const double *corr, int64_t n_rows, int64_t n_cols,
                                double u0, double v0, double pitch, double sdd, double sod,
                                double cphi, double sphi, const double *rot,
                                const double *tvec, double radius, double height, int64_t nh,
                                int64_t nt, int64_t nr, double *num, double *den) {
    const double dr = radius / (double)nr;
    const double dth = OR_TWO_PI / (double)nt;
    const double dh = height / (double)nh;
    const double half_h = 0.5 * height;
    const double depth_floor = 1e-6 * sod;
    (void)nh;
    int64_t k = m / (nt * nr);
    int64_t j = (m / nr) % nt;
    int64_t ir = m % nr;
    double r = ((double)ir + 0.5) * dr;
    double th = ((double)j + 0.5) * dth;
    double h = ((double)k + 0.5) * dh - half_h;
    double xo = r * cos(th);
    double yo = r * sin(th);
    double xw = rot[0] * xo + rot[1] * yo + rot[2] * h + tvec[0];
    double yw = rot[3] * xo + rot[4] * yo + rot[5] * h + tvec[1];
    double zw = rot[6] * xo + rot[7] * yo + rot[8] * h + tvec[2];
    double xi = cphi * xw - sphi * yw;
    double yi = sphi * xw + cphi * yw;
    double depth = sod + yi;
    if (depth <= depth_floor) return;
    double scale = sdd / (depth * pitch);
    double a, b;
    bilinear_gather(corr, n_rows, n_cols, u0 + xi * scale, v0 + zw * scale, &a, &b);
    *num += a;
    *den += b;
}

/* _kernels.py:380-417 -- voxel-driven BP; ACCUMULATES into num/den. */
void oracle_backproject_cyl(const double *corr, int64_t n_rows, int64_t n_cols, double u0,
                            double v0, double pitch, double sdd, double sod, double cphi,
                            double sphi, const double *rot, const double *tvec,
                            double radius, double height, int64_t nh, int64_t nt,
                            int64_t nr, double *num, double *den) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < nh * nt * nr; ++m)
        bp_cyl_voxel(m, corr, n_rows, n_cols, u0, v0, pitch, sdd, sod, cphi, sphi, rot, tvec,
                     radius, height, nh, nt, nr, &num[m], &den[m]);
}

/* The same per-voxel function on an explicit voxel list (flat indices
 * idx[0..n_idx)); num/den have n_idx entries (accumulated).  For parity at
 * sizes where the whole-volume BP is too slow for a test. */
void oracle_backproject_cyl_voxels(const double *corr, int64_t n_rows, int64_t n_cols,
                                   double u0, double v0, double pitch, double sdd, double sod,
                                   double cphi, double sphi, const double *rot,
                                   const double *tvec, double radius, double height,
                                   int64_t nh, int64_t nt, int64_t nr, const int64_t *idx,
                                   int64_t n_idx, double *num, double *den) {
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < n_idx; ++q)
        bp_cyl_voxel(idx[q], corr, n_rows, n_cols, u0, v0, pitch, sdd, sod, cphi, sphi, rot,
                     tvec, radius, height, nh, nt, nr, &num[q], &den[q]);
}

/* _kernels.py:420-443 -- one voxel of the Cartesian BP. */
static inline void bp_cart_voxel(int64_t m, const double *corr, int64_t n_rows, int64_t n_cols,
                                 double u0, double v0, double pitch, double sdd, double sod,
                                 double cphi, double sphi, double vs, double ox, double oy,
                                 double oz, int64_t ny, int64_t nx, double *num, double *den) {
    const double depth_floor = 1e-6 * sod;
    int64_t k = m / (ny * nx);
    int64_t j = (m / nx) % ny;
    int64_t i = m % nx;
    double xw = ox + ((double)i + 0.5) * vs;
    double yw = oy + ((double)j + 0.5) * vs;
    double zw = oz + ((double)k + 0.5) * vs;
    double xi = cphi * xw - sphi * yw;
    double yi = sphi * xw + cphi * yw;
    double depth = sod + yi;
    if (depth <= depth_floor) return;
    double scale = sdd / (depth * pitch);
    double a, b;
    bilinear_gather(corr, n_rows, n_cols, u0 + xi * scale, v0 + zw * scale, &a, &b);
    *num += a;
    *den += b;
}

/* _kernels.py:420-443 */
void oracle_backproject_cart(const double *corr, int64_t n_rows, int64_t n_cols, double u0,
                             double v0, double pitch, double sdd, double sod, double cphi,
                             double sphi, double vs, double ox, double oy, double oz,
                             int64_t nz, int64_t ny, int64_t nx, double *num, double *den) {
#pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < nz * ny * nx; ++m)
        bp_cart_voxel(m, corr, n_rows, n_cols, u0, v0, pitch, sdd, sod, cphi, sphi, vs, ox, oy,
                      oz, ny, nx, &num[m], &den[m]);
}

void oracle_backproject_cart_voxels(const double *corr, int64_t n_rows, int64_t n_cols,
                                    double u0, double v0, double pitch, double sdd, double sod,
                                    double cphi, double sphi, double vs, double ox, double oy,
                                    double oz, int64_t nz, int64_t ny, int64_t nx,
                                    const int64_t *idx, int64_t n_idx, double *num,
                                    double *den) {
    (void)nz;
#pragma omp parallel for schedule(static)
    for (int64_t q = 0; q < n_idx; ++q)
        bp_cart_voxel(idx[q], corr, n_rows, n_cols, u0, v0, pitch, sdd, sod, cphi, sphi, vs, ox,
                      oy, oz, ny, nx, &num[q], &den[q]);
}

/* Threads the OpenMP runtime will use (for the cpu_baseline's "cores"). */
int oracle_max_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}
