/*
 * cyltomo_b200.h -- C-ABI of the B200-native cone-beam projector / SART path.
 *
 * Drop-in seam: the reference's kernel boundary is the set of numba kernels
 * in cyltomo/_kernels.py, called with plain arrays and scalars by
 * cyltomo/projector.py and cyltomo/grid.py.  Every entry point below replaces
 * one of them (file:line cited per function) or fuses a reference numpy step
 * (cyltomo/recon.py) into a kernel epilogue.
 *
 * Conventions
 *  - All array arguments are DEVICE pointers owned by the caller, float32
 *    unless stated (the reference is float64 on the host; the B200 path keeps
 *    fp32 data and does per-ray setup in fp64 -- see DESIGN.md "Numerics").
 *  - Cylindrical volumes: mu[n_h][n_theta][n_r], r fastest
 *    (cyltomo/grid.py:91-93).  Cartesian volumes: mu[n_z][n_y][n_x].
 *  - Projection stacks / correction images: [views][det_rows][det_cols].
 *  - Struct arguments passed by pointer are HOST pointers, read during the
 *    call only.  `views`/`dets` tables are DEVICE arrays (upload once per
 *    geometry; that keeps every call capturable in a CUDA graph).
 *  - `stream` is a cudaStream_t (NULL = legacy default stream).  Calls are
 *    asynchronous; no call synchronises the device.
 *  - Return value: CT_OK or a negative CT_ERR_*; CT_ERR_CUDA means a launch
 *    failed -- ct_last_error() gives the CUDA error string.  No exceptions
 *    cross the ABI.
 *  - FP entry points OVERWRITE their outputs; BP entry points accumulate or
 *    overwrite as documented (the reference's backproject_* accumulate).
 *  - Results are deterministic: no atomics on data, fixed reduction order.
 */
#ifndef CYLTOMO_B200_H
#define CYLTOMO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CT_ABI_VERSION 9

#define CT_OK 0
#define CT_ERR_ARG (-1)   /* invalid argument (null pointer, bad size) */
#define CT_ERR_CUDA (-2)  /* kernel launch / runtime failure */

typedef void *ct_stream_t; /* cudaStream_t */

/* Object-aligned cylindrical grid (cyltomo/grid.py:62-110).  rot is the
 * row-major object->world rotation R, t the translation (X' = R X + t). */
typedef struct ct_cyl_grid {
    int32_t n_h, n_theta, n_r, _pad;
    double radius, height;
    double rot[9];
    double t[3];
} ct_cyl_grid;

/* World-aligned Cartesian grid (cyltomo/grid.py:139-187). */
typedef struct ct_cart_grid {
    int32_t n_z, n_y, n_x, _pad;
    double voxel_size;
    double origin[3];
} ct_cart_grid;

/* Per-view ray basis for the forward projector: source, pixel-(0,0) centre,
 * per-column and per-row steps.  For cylindrical grids these are already in
 * the grid-aligned frame (cyltomo/projector.py:83-88); for Cartesian grids
 * they are world-frame (cyltomo/geometry.py:257-273). */
typedef struct ct_ray_view {
    double src[3], origin[3], du[3], dv[3];
} ct_ray_view;

/* Per-view detector parameters for the back-projector
 * (cyltomo/projector.py:151-163): principal point, pitch, distances and the
 * cos/sin of the stage angle. */
typedef struct ct_det_view {
    double u0, v0, pitch, sdd, sod, cphi, sphi, _pad;
} ct_det_view;

/* Ray sampling (cyltomo/projector.py:28-56): step in mm (already resolved),
 * supersample >= 1, nearest != 0 for nearest-neighbour interpolation. */
typedef struct ct_sampling {
    double step;
    int32_t supersample;
    int32_t nearest;
} ct_sampling;

/* Fused SART update (cyltomo/recon.py:105-119):
 *   touched = den > 0 [&& weights != 0]
 *   mu[touched] = max(mu + relaxation * w * num / den, 0 if nonneg)
 * weights may be NULL (unweighted). */
typedef struct ct_update {
    float relaxation;
    int32_t nonneg;
    const float *weights;
    float *mu;
    /* (ABI v6) peer-store all-gather fused into the update: when n_peers > 0,
     * every updated voxel is also stored into each of the n_peers replica
     * volumes mu_peers[p] (device array of device pointers, e.g. the
     * symmetric-memory buffers of the ranks, NVLink P2P stores) instead of
     * only into mu. */
    float *const *mu_peers;
    int32_t n_peers;
    int32_t _pad;
    /* (ABI v9) NULL, or a device int64 array [n_peers][2]: voxel m goes to
     * replica p only when peer_ranges[2p] <= m < peer_ranges[2p+1] (the
     * slab decomposition's halo layers, slab.SlabSartRun fused mode). */
    const int64_t *peer_ranges;
} ct_update;

/* Detector / batch description shared by the batched calls:
 * view_ids[b] (device, int32) is the global view index of batch slot b; it
 * selects the entry of `views`/`dets`, of `p_meas` ([P][rows][cols]) and of
 * `row_thr`.  view_ids may be NULL, meaning slot b == view b. */
typedef struct ct_batch {
    int32_t n_batch;
    int32_t det_rows, det_cols;
    int32_t _pad;
    const int32_t *view_ids;
} ct_batch;

/* ---- library ------------------------------------------------------------ */
int ct_abi_version(void);
const char *ct_last_error(void);
/* Compiled-for architecture string, e.g. "sm_100a". */
const char *ct_arch(void);

/* ---- forward projection (cyltomo/_kernels.py:238-293 forward_cyl,
 *      :296-343 forward_cart) ---------------------------------------------- */

/* `gather` (optional, may be NULL): the gather layout of the same mu built by
 * ct_pack_gather_* (8 floats per cell: the trilinear polynomial of its 2x2x2
 * neighbourhood, one 32-byte sector).  With it every FP sample is one 32-byte
 * load instead of eight scattered 4-byte loads; results are identical.
 * It must be rebuilt after mu changes. */

/* forward_cyl over a batch of views: out_p / out_w are [n_batch][rows][cols]
 * (OVERWRITTEN).  out_w = in-support sample count * step / ss^2 (the SART row
 * sums, cyltomo/projector.py:100-103); out_w may be NULL. */
int ct_fp_cyl(const float *mu, const float *gather, const ct_cyl_grid *grid, const ct_ray_view *views,
              const ct_batch *batch, const ct_sampling *sampling,
              float *out_p, float *out_w, ct_stream_t stream);

int ct_fp_cart(const float *mu, const float *gather, const ct_cart_grid *grid, const ct_ray_view *views,
               const ct_batch *batch, const ct_sampling *sampling,
               float *out_p, float *out_w, ct_stream_t stream);

/* FP with the SART correction epilogue (cyltomo/recon.py:96-102):
 *   corr[b] = (w > row_thr[v]) ? (p_meas[v] - sim) / w : 0,   v = view_ids[b]
 * row_thr (device, float64, [P]) = ROW_SUM_SKIP_FRACTION * max_row per view
 * (ct_rowsum_max_*).  corr is [n_batch][rows][cols]. */
int ct_fp_cyl_correction(const float *mu, const float *gather, const ct_cyl_grid *grid, const ct_ray_view *views,
                         const ct_batch *batch, const ct_sampling *sampling,
                         const float *p_meas, const double *row_thr, float *corr,
                         ct_stream_t stream);
int ct_fp_cart_correction(const float *mu, const float *gather, const ct_cart_grid *grid, const ct_ray_view *views,
                          const ct_batch *batch, const ct_sampling *sampling,
                          const float *p_meas, const double *row_thr, float *corr,
                          ct_stream_t stream);

/* FP with the residual epilogue (cyltomo/recon.py:148-153): adds
 * sum_b sum_pix (p_meas[v] - sim)^2 (fp64, fixed reduction order) into
 * *accum (device double).  `scratch` must hold ct_residual_scratch_len()
 * doubles. */
int64_t ct_residual_scratch_len(const ct_batch *batch);
int ct_fp_cyl_residual(const float *mu, const float *gather, const ct_cyl_grid *grid, const ct_ray_view *views,
                       const ct_batch *batch, const ct_sampling *sampling,
                       const float *p_meas, double *scratch, double *accum,
                       ct_stream_t stream);
int ct_fp_cart_residual(const float *mu, const float *gather, const ct_cart_grid *grid, const ct_ray_view *views,
                        const ct_batch *batch, const ct_sampling *sampling,
                        const float *p_meas, double *scratch, double *accum,
                        ct_stream_t stream);

/* Row ranges and residual slots (ABI v6), for work split across launches and
 * ranks (SART residual deferral, recon.py; angle sharding, distributed.py).
 *  - Rows: the batch's rays are numbered by flattened row f = b * det_rows +
 *    row; only rows in [row_lo, row_hi) are marched, and the correction of
 *    row f lands at corr[(f - row_lo) * det_cols + col].
 *  - Residual slots: block partials land where an identity-ordered batch of
 *    n_slots views (view_ids 0..n_slots-1) would put them, so launches over
 *    disjoint views / row ranges aligned to ct_fp_row_tile() fill one
 *    scratch (ct_residual_scratch_len of an n_slots batch) whose
 *    ct_residual_sum is bit-identical to ct_fp_*_residual over all n_slots
 *    views.  batch->view_ids is required with a scratch.
 *  - ct_fp_*_correction_rows: the correction epilogue of ct_fp_*_correction;
 *    with a scratch also the residual partials of the same simulation (the
 *    residual FP of pass k and the first subset's correction FP of pass k+1
 *    read the same mu, recon.py:171-181 / PAPER.md:182-187); with
 *    n_peers > 0 each correction is stored at corr_peers[p][peer_offset +
 *    (f - row_lo) * det_cols + col] for every p instead of into corr (the
 *    all-gather of the corrections fused into the FP: NVLink P2P stores);
 *  - ct_fp_*_residual_rows: residual partials only (no sum);
 *  - ct_residual_sum: *accum += fixed-order sum of scratch[0..n);
 *  - ct_fp_row_tile: rows per FP block for this detector. */
int ct_fp_row_tile(const ct_batch *batch);
int ct_fp_cyl_correction_rows(const float *mu, const float *gather, const ct_cyl_grid *grid,
                              const ct_ray_view *views, const ct_batch *batch,
                              const ct_sampling *sampling, const float *p_meas,
                              const double *row_thr, float *corr, int64_t row_lo,
                              int64_t row_hi, int n_slots, double *scratch,
                              float *const *corr_peers, int n_peers, int64_t peer_offset,
                              ct_stream_t stream);
int ct_fp_cart_correction_rows(const float *mu, const float *gather, const ct_cart_grid *grid,
                               const ct_ray_view *views, const ct_batch *batch,
                               const ct_sampling *sampling, const float *p_meas,
                               const double *row_thr, float *corr, int64_t row_lo,
                               int64_t row_hi, int n_slots, double *scratch,
                               float *const *corr_peers, int n_peers, int64_t peer_offset,
                               ct_stream_t stream);
int ct_fp_cyl_residual_rows(const float *mu, const float *gather, const ct_cyl_grid *grid,
                            const ct_ray_view *views, const ct_batch *batch,
                            const ct_sampling *sampling, const float *p_meas, int64_t row_lo,
                            int64_t row_hi, int n_slots, double *scratch, ct_stream_t stream);
int ct_fp_cart_residual_rows(const float *mu, const float *gather, const ct_cart_grid *grid,
                             const ct_ray_view *views, const ct_batch *batch,
                             const ct_sampling *sampling, const float *p_meas, int64_t row_lo,
                             int64_t row_hi, int n_slots, double *scratch, ct_stream_t stream);
int ct_residual_sum(const double *scratch, int64_t n, double *accum, ct_stream_t stream);

/* Row bands (ABI v8; the slab decomposition of distributed.SlabSartRun): per
 * view slot b, only detector rows [bands[2b], bands[2b+1]) are marched.
 * bands is a DEVICE int32 array [n_batch][2]; every bands[2b] must be a
 * multiple of ct_fp_row_tile() and band_rows >= max(bands[2b+1] - bands[2b]).
 * Outputs land at their full-stack positions: the correction of (b, row,
 * col) at corr[(b * det_rows + row) * det_cols + col] (rows outside the band
 * untouched); residual partials at the n_slots-view slots of the full launch
 * (see above), so disjoint bands of one view on different ranks fill
 * disjoint slots.  _correction_bands with a scratch: both epilogues.
 * (ABI v9) corr_peers / n_peers: the corrections are stored into every
 * corr_peers[p] at the same full-stack position instead of into corr, and,
 * with peer_rows (device int32 [n_batch][n_peers][2]) set, into replica p
 * only for rows peer_rows[2 (b n_peers + p)] <= row < peer_rows[... + 1]:
 * the exchange of the slab decomposition fused into the FP (NVLink peer
 * stores into symmetric memory). */
int ct_fp_cyl_correction_bands(const float *mu, const float *gather, const ct_cyl_grid *grid,
                               const ct_ray_view *views, const ct_batch *batch,
                               const ct_sampling *sampling, const float *p_meas,
                               const double *row_thr, float *corr, const int32_t *bands,
                               int band_rows, int n_slots, double *scratch,
                               float *const *corr_peers, int n_peers,
                               const int32_t *peer_rows,
                               ct_stream_t stream);
int ct_fp_cart_correction_bands(const float *mu, const float *gather, const ct_cart_grid *grid,
                                const ct_ray_view *views, const ct_batch *batch,
                                const ct_sampling *sampling, const float *p_meas,
                                const double *row_thr, float *corr, const int32_t *bands,
                                int band_rows, int n_slots, double *scratch,
                               float *const *corr_peers, int n_peers,
                               const int32_t *peer_rows,
                                ct_stream_t stream);
int ct_fp_cyl_residual_bands(const float *mu, const float *gather, const ct_cyl_grid *grid,
                             const ct_ray_view *views, const ct_batch *batch,
                             const ct_sampling *sampling, const float *p_meas,
                             const int32_t *bands, int band_rows, int n_slots, double *scratch,
                             ct_stream_t stream);
int ct_fp_cart_residual_bands(const float *mu, const float *gather, const ct_cart_grid *grid,
                              const ct_ray_view *views, const ct_batch *batch,
                              const ct_sampling *sampling, const float *p_meas,
                              const int32_t *bands, int band_rows, int n_slots,
                              double *scratch, ct_stream_t stream);
/* Geometry only (ABI v8): per (view slot b, detector row) the smallest and
 * largest FP cell layer kc any sample of the row's rays reads, cells[2 *
 * (b * det_rows + row) + {0, 1}] (device int32, overwritten; rows without
 * samples: INT32_MAX, INT32_MIN).  kc is the march's own fp32 h (z) cell
 * index: the FP reads mu layers kc - 1 and kc (clamped to the grid) there,
 * i.e. gather cells packed by ct_pack_gather_*_layers(kc_lo, kc_hi). */
int ct_row_cells_cyl(const ct_cyl_grid *grid, const ct_ray_view *views, const ct_batch *batch,
                     const ct_sampling *sampling, int32_t *cells, ct_stream_t stream);
int ct_row_cells_cart(const ct_cart_grid *grid, const ct_ray_view *views, const ct_batch *batch,
                      const ct_sampling *sampling, int32_t *cells, ct_stream_t stream);

/* Geometry-only in-support sample count summed per detector row:
 * row_samples[b * det_rows + row] (uint64, overwritten), the per-row cost
 * model of the angle-sharded row split (distributed.py; ABI v6). */
int ct_row_samples_cyl(const ct_cyl_grid *grid, const ct_ray_view *views, const ct_batch *batch,
                       const ct_sampling *sampling, uint64_t *row_samples, ct_stream_t stream);
int ct_row_samples_cart(const ct_cart_grid *grid, const ct_ray_view *views,
                        const ct_batch *batch, const ct_sampling *sampling,
                        uint64_t *row_samples, ct_stream_t stream);

/* Geometry-only row-sum maximum per view (the max_row of
 * cyltomo/recon.py:96-98), computed without marching: max_row[b] (device,
 * float64, [n_batch]) = max over pixels of out_w.  Exact (sample counts are
 * computed with the reference's fp64 interval arithmetic). */
int ct_rowsum_max_cyl(const ct_cyl_grid *grid, const ct_ray_view *views,
                      const ct_batch *batch, const ct_sampling *sampling,
                      double *max_row, ct_stream_t stream);
int ct_rowsum_max_cart(const ct_cart_grid *grid, const ct_ray_view *views,
                       const ct_batch *batch, const ct_sampling *sampling,
                       double *max_row, ct_stream_t stream);

/* ---- back-projection (cyltomo/_kernels.py:380-417 backproject_cyl,
 *      :420-443 backproject_cart) ----------------------------------------- */

/* Sum over the batch of backproject_*(corr[b], view_ids[b]).  accumulate != 0
 * adds into num/den (the reference's semantics); 0 overwrites.  den may be
 * NULL.  trig (device, float64, [2*n_theta]) holds cos(theta_j), sin(theta_j)
 * of the voxel centres (see ct_cyl_trig).
 * `quads` (optional, may be NULL): the bilinear footprints of the same corr
 * stack built by ct_pack_quads; with it an interior voxel-view reads one
 * 16-byte footprint instead of four scattered taps.  Results are identical
 * to within fp32 rounding of the bilinear form (same taps, same weights).
 * n_batch * det_rows * det_cols must be < 2^32. */
int ct_bp_cyl(const float *corr, const float *quads, const ct_det_view *dets,
              const ct_batch *batch, const ct_cyl_grid *grid, const double *trig, float *num,
              float *den, int accumulate, ct_stream_t stream);
int ct_bp_cart(const float *corr, const float *quads, const ct_det_view *dets,
               const ct_batch *batch, const ct_cart_grid *grid, float *num, float *den,
               int accumulate, ct_stream_t stream);

/* BP of the batch followed by the fused SART / OS-SART update of
 * cyltomo/recon.py:105-119 with num/den = the batch sums (kept in registers). */
int ct_bp_cyl_update(const float *corr, const float *quads, const ct_det_view *dets,
                     const ct_batch *batch, const ct_cyl_grid *grid, const double *trig,
                     const ct_update *upd, ct_stream_t stream);
int ct_bp_cart_update(const float *corr, const float *quads, const ct_det_view *dets,
                      const ct_batch *batch, const ct_cart_grid *grid, const ct_update *upd,
                      ct_stream_t stream);

/* Bilinear footprints of a correction stack [n_batch][rows][cols]: quad
 * (b, v, u) = (c[v][u], c[v][u+1], c[v+1][u], c[v+1][u+1]) of image b (0 past
 * the last row / column), 4 floats per pixel, 16-byte aligned.
 * ct_quads_floats gives the buffer length in floats. */
int64_t ct_quads_floats(const ct_batch *batch);
int ct_pack_quads(const float *corr, const ct_batch *batch, float *quads, ct_stream_t stream);

/* Fill trig[0:n] = cos((j+.5)dtheta), trig[n:2n] = sin(...) (fp64). */
/* Fused BP + SART update restricted to voxels [offset, offset+count) of the
 * flat [n_h][n_theta][n_r] (or [n_z][n_y][n_x]) volume: a rank's shard in
 * the angle-sharded OS-SART (distributed.py); every voxel's result equals
 * ct_bp_*_update's (ABI v6). */
int ct_bp_cyl_update_range(const float *corr, const float *quads, const ct_det_view *dets,
                           const ct_batch *batch, const ct_cyl_grid *grid, const double *trig,
                           const ct_update *upd, int64_t offset, int64_t count,
                           ct_stream_t stream);
int ct_bp_cart_update_range(const float *corr, const float *quads, const ct_det_view *dets,
                            const ct_batch *batch, const ct_cart_grid *grid,
                            const ct_update *upd, int64_t offset, int64_t count,
                            ct_stream_t stream);

int ct_cyl_trig(const ct_cyl_grid *grid, double *trig, ct_stream_t stream);

/* Stand-alone update from reduced num/den over voxels [offset, offset+count)
 * (the multi-GPU path: BP partials -> NCCL reduce-scatter -> this).  Writes
 * upd->mu only: upd->n_peers must be 0 (CT_ERR_ARG otherwise).  Every entry
 * point taking a ct_update rejects n_peers < 0 and n_peers > 0 with a null
 * mu_peers. */
int ct_sart_update(const float *num, const float *den, int64_t offset, int64_t count,
                   const ct_update *upd, ct_stream_t stream);

/* ---- gather layout for the forward projector ------------------------------ */
/* Number of floats of the gather buffer: 8 per cell, cells (n_h+1, n_theta+1,
 * n_r+1) for a cylindrical grid, (n_z+1, n_y+1, n_x+1) for a Cartesian one,
 * r (x) fastest; each h (z) layer is padded by < 256 cells so that the cell
 * index needs no bias term. */
int64_t ct_gather_floats_cyl(const ct_cyl_grid *grid);
int64_t ct_gather_floats_cart(const ct_cart_grid *grid);
/* (ABI v7) Which gather layout ct_pack_gather_* builds for this grid (and the
 * FP reads): CT_GL_OCT linear 32-byte trilinear cells, CT_GL_QUAD bricked
 * 16-byte bilinear layer cells (layers > 10 MB), CT_GL_OCTB 32-byte cells in
 * 2x2 bricks (layers > 6 MB); < 0 for a bad grid.  Tests use it to prove
 * which production path a parity case exercised. */
#define CT_GL_OCT 1
#define CT_GL_QUAD 2
#define CT_GL_OCTB 3
int ct_gather_layout_cyl(const ct_cyl_grid *grid);
int ct_gather_layout_cart(const ct_cart_grid *grid);
/* Cell (kc, jc, ic) holds the trilinear corner (k, j, i) = (kc-1, jc-1, ic-1)
 * with a one-cell halo at index -1 (r/h: a copy of index 0; theta: the wrapped
 * row n_theta-1) as the coefficients of
 *   f(wr, wt, wh) = c0 + cr wr + ct wt + crt wr wt + ch wh + crh wr wh + cth wt wh
 *                   + crth wr wt wh,
 * stored (c0, cr, ct, crt, ch, crh, cth, crth), of the 8 corner values
 * mu(k+X, j+Y, i+Z) (r/h clamp to the grid, theta wraps; Cartesian: y plays
 * theta's role and all three axes clamp).  16-byte aligned. */
int ct_pack_gather_cyl(const float *mu, const ct_cyl_grid *grid, float *gather,
                       ct_stream_t stream);
int ct_pack_gather_cart(const float *mu, const ct_cart_grid *grid, float *gather,
                        ct_stream_t stream);
/* (ABI v8) Pack only what FP cell layers kc in [kc_lo, kc_hi] read (see
 * ct_row_cells_*; reads mu layers kc_lo - 1 .. kc_hi, clamped); the rest of
 * the buffer is left as is.  ct_pack_gather_* = kc in [0, n_h] ([0, n_z]). */
int ct_pack_gather_cyl_layers(const float *mu, const ct_cyl_grid *grid, float *gather,
                              int32_t kc_lo, int32_t kc_hi, ct_stream_t stream);
int ct_pack_gather_cart_layers(const float *mu, const ct_cart_grid *grid, float *gather,
                               int32_t kc_lo, int32_t kc_hi, ct_stream_t stream);

/* ---- input conversion (cyltomo/projector.py:169-181) ---------------------- */
/* out[i] = -ln(intensity[i] / I0) with I0 = flat[i % npix] (flat != NULL, one
 * image broadcast over the views) or flat_scalar.  Computed in fp64 from the
 * fp32 inputs.  If any I <= 0 or I0 <= 0, *bad (device int, caller-zeroed) is
 * set to 1 (the reference raises NonPositiveIntensity). */
int ct_line_integrals(const float *intensity, int64_t n, int64_t npix, const float *flat,
                      double flat_scalar, float *out, int *bad, ct_stream_t stream);

/* ---- point sampling (cyltomo/_kernels.py:154-163, grid.py:261-319) ------- */
int ct_sample_cyl(const float *mu, const ct_cyl_grid *grid, const double *rs,
                  const double *ths, const double *hs, int64_t n, int nearest,
                  float *out, ct_stream_t stream);
int ct_sample_cart(const float *mu, const ct_cart_grid *grid, const double *xs,
                   const double *ys, const double *zs, int64_t n, int nearest,
                   float *out, ct_stream_t stream);
/* resample_cyl_to_cyl (cyltomo/grid.py:310-319): evaluate src at every voxel
 * centre of dst (both in object coordinates; poses ignored). */
int ct_resample_cyl_to_cyl(const float *src_mu, const ct_cyl_grid *src,
                           const ct_cyl_grid *dst, int nearest, float *dst_mu,
                           ct_stream_t stream);

/* ---- projection-image statistics for the pose step (cyltomo/imgproc.py) ---- */
/* Per-view min / max of images[n_views][npix] (mn, mx: device float[n_views]). */
int ct_image_minmax(const float *images, int n_views, int64_t npix, float *mn, float *mx,
                    ct_stream_t stream);
/* np.histogram(view, bins, range=(lo[v], hi[v])) per view, same fp64 binning
 * and edge corrections as numpy's uniform-bin path; counts[n_views][bins]. */
int ct_image_histogram(const float *images, int n_views, int64_t npix, const double *lo,
                       const double *hi, int bins, unsigned *counts, ct_stream_t stream);
/* mask[v] = dilate(images[v] > levels[v], square of half-width radius) (uint8). */
int ct_threshold_dilate(const float *images, int n_views, int rows, int cols,
                        const double *levels, int radius, unsigned char *mask,
                        ct_stream_t stream);
/* Per view and row: leftmost / rightmost column of mask & ~remove outside the
 * n_rects (row0, row1, col0, col1) half-open rectangles; -1 when empty.
 * remove and rects may be NULL.  left/right: int[n_views][rows]. */
int ct_row_extents(const unsigned char *mask, const unsigned char *remove, int n_views,
                   int rows, int cols, const int *rects, int n_rects, int *left, int *right,
                   ct_stream_t stream);
/* Fused threshold + extents for a ladder of n_levels (<= 16) thresholds per
 * view (levels[n_views][n_levels], foreground = image > level) in one pass;
 * left/right: int[n_levels][n_views][rows]. */
int ct_row_extents_levels(const float *images, const double *levels, int n_levels,
                          const unsigned char *remove, int n_views, int rows, int cols,
                          const int *rects, int n_rects, int *left, int *right,
                          ct_stream_t stream);
/* Axis endpoints (cyltomo/imgproc.py:97-131 band-corner rule) of n_tables
 * extent tables left/right[n_tables][rows] (as ct_row_extents writes them):
 * out[t] = (top_u, top_v, bottom_u, bottom_v) with top above bottom,
 * status[t] = 0 ok, 1 empty mask, 2 fewer than two rows. */
int ct_axis_endpoints(const int *left, const int *right, int n_tables, int rows, int band,
                      double *out, int *status, ct_stream_t stream);
/* Mean bilinear grey value of a strip parallel to each view's projected axis
 * (axes[v] = u_top, v_top, u_bottom, v_bottom, |bottom - top|), signed offset / width in
 * pixels (cyltomo/imgproc.py:152-180); out[v] = NaN if the strip is off-frame. */
int ct_strip_profiles(const float *images, int n_views, int rows, int cols, const double *axes,
                      double offset, double width, double *out, ct_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* CYLTOMO_B200_H */
