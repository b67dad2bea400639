"""Would TMA staging of the BP's footprints (north_star: "shared-memory/TMA
staging of projection rows") move fewer bytes through the SM's L1/shared
SRAM than the current L1-cached gathers?  Host-side geometry estimate.

For a sample of BP CTA tiles (64 r-voxels x 4 theta rows at one h layer, as
bp_kernel<BP_PR=8>) and views of C2 and C5, project the tile's voxels
(cyltomo/_kernels.py:396-414 arithmetic, numpy fp64) and report:
  * the tile's footprint bounding box (u, v extent in pixels, +1 for the
    bilinear taps) -- the smallest rectangle a TMA tile load must bring into
    shared memory, and its bytes with 16-byte footprint quads;
  * the distinct quads the tile actually reads (the useful bytes);
  * the bytes the current kernel moves through the L1 data pipe for the same
    (tile, view): 8 warps x wavefronts per request x 128 B, with the
    measured 10.0 (C2) / 11.1 (C5) wavefronts per request
    (profiles/r02_ncu_c2.txt, r02_ncu_c5.txt).
Staging wins only if the window fill (written into shared memory) plus the
shared-memory reads (>= 4 wavefronts per warp request) is below that.
"""
import math
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2005_11976_b200 import workloads as W  # noqa: E402

WF_PER_REQ = {"c2": 10.04, "c5": 11.1}


def tile_stats(wl, n_tiles=400, seed=0):
    g, geom = wl.grid, wl.geom
    rng = np.random.default_rng(seed)
    R = np.asarray(g.rotation, dtype=float)
    t = np.asarray(g.pose.t, dtype=float)
    dr, dth, dh = g.radius / g.n_r, 2 * math.pi / g.n_theta, g.height / g.n_h
    u0, v0 = geom.principal_point
    out = []
    for _ in range(n_tiles):
        k = rng.integers(g.n_h)
        j0 = rng.integers(g.n_theta // 4) * 4
        i0 = rng.integers(g.n_r // 64) * 64
        view = rng.integers(geom.n_proj)
        ir, jj = np.meshgrid(np.arange(i0, i0 + 64), np.arange(j0, j0 + 4))
        r = (ir + 0.5) * dr
        th = (jj + 0.5) * dth
        h = (k + 0.5) * dh - 0.5 * g.height
        obj = np.stack([r * np.cos(th), r * np.sin(th), np.full_like(r, h)], -1).reshape(-1, 3)
        w = obj @ R.T + t
        phi = geom.stage_angles[view]
        c, s = math.cos(phi), math.sin(phi)
        xi = c * w[:, 0] - s * w[:, 1]
        yi = s * w[:, 0] + c * w[:, 1]
        scale = geom.sdd / ((geom.sod + yi) * geom.pixel_pitch)
        u = u0 + xi * scale
        v = v0 + w[:, 2] * scale
        iu, iv = np.floor(u).astype(int), np.floor(v).astype(int)
        bbox = (iu.max() - iu.min() + 2) * (iv.max() - iv.min() + 2)
        distinct = len(set(zip(iu.tolist(), iv.tolist())))
        out.append((iu.max() - iu.min() + 2, iv.max() - iv.min() + 2, bbox, distinct))
    return np.array(out, dtype=float)


def main():
    for name, wl in (("c2", W.c2_medium()), ("c5", W.c5_object(0))):
        st = tile_stats(wl)
        bu, bv, bbox, distinct = st.T
        tma_bytes = 16 * bbox
        smem_read = 8 * 4 * 128                  # >= 4 wavefronts per 128-bit warp request
        l1_bytes = 8 * WF_PER_REQ[name] * 128
        print(f"{name}: window u {np.median(bu):.0f} (p95 {np.percentile(bu, 95):.0f}) x v "
              f"{np.median(bv):.0f} (p95 {np.percentile(bv, 95):.0f}) px; bbox "
              f"{np.median(bbox):.0f} quads, distinct {np.median(distinct):.0f} quads "
              f"({np.median(distinct / bbox) * 100:.0f} % of the window)")
        print(f"    per (CTA, view): exact-bbox window fill {np.median(tma_bytes) / 1024:.1f} KiB + "
              f"shared reads >= {smem_read / 1024:.1f} KiB  vs  current L1 data-pipe "
              f"{l1_bytes / 1024:.1f} KiB (8 warps x {WF_PER_REQ[name]} wavefronts x 128 B)")
        # a TMA tile load moves its whole (fixed) box: one box covering the
        # p99 window, or the window tiled by 16 x 4-quad boxes
        p99u, p99v = np.percentile(bu, 99), np.percentile(bv, 99)
        box = 16 * (8 * math.ceil(p99u / 8)) * (4 * math.ceil(p99v / 4))
        tiled = 16 * 64 * np.ceil(bu / 16) * np.ceil(bv / 4)
        print(f"    fixed box for the p99 window ({p99u:.0f} x {p99v:.0f}): {box / 1024:.1f} KiB "
              f"per (CTA, view); 16x4-quad tiles: {np.median(tiled) / 1024:.1f} KiB median "
              f"({np.median(np.ceil(bu / 16) * np.ceil(bv / 4)):.0f} TMA ops)")


if __name__ == "__main__":
    main()
