"""The C-ABI library: loads without a GPU, exports every declared symbol, struct
layouts agree with include/cyltomo_b200.h, and the product refuses to fall back
to the CPU."""

import ctypes as C
import re
import subprocess
import textwrap
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "cyltomo_b200.h"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(ct_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_2005_11976_b200 import _native as N
    lib = N.load_library()
    names = declared_functions()
    assert len(names) >= 20
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) == set(N.EXPORTED_SYMBOLS)
    assert lib.ct_abi_version() == N.CT_ABI_VERSION
    assert lib.ct_arch() == b"sm_100a"


def test_nm_shows_extern_c_symbols():
    from paper_2005_11976_b200 import _native as N
    out = subprocess.run(["nm", "-D", "--defined-only", str(N.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r" T (ct_\w+)", out))
    assert set(declared_functions()) <= exported


def test_struct_layouts_match_header(tmp_path):
    """Compile a C probe against the header and compare sizeof/offsetof with ctypes."""
    from paper_2005_11976_b200 import _native as N
    probe = tmp_path / "probe.c"
    probe.write_text(textwrap.dedent("""
        #include <stdio.h>
        #include <stddef.h>
        #include "cyltomo_b200.h"
        int main(void) {
          printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(ct_cyl_grid), sizeof(ct_cart_grid),
                 sizeof(ct_ray_view), sizeof(ct_det_view), sizeof(ct_sampling),
                 sizeof(ct_update), sizeof(ct_batch));
          printf("%zu %zu %zu %zu %zu %zu %zu\\n", offsetof(ct_cyl_grid, rot),
                 offsetof(ct_cyl_grid, t), offsetof(ct_update, weights),
                 offsetof(ct_batch, view_ids), offsetof(ct_update, mu_peers),
                 offsetof(ct_update, n_peers), offsetof(ct_update, peer_ranges));
          return 0;
        }"""))
    exe = tmp_path / "probe"
    cc = "/usr/bin/gcc" if Path("/usr/bin/gcc").exists() else "gcc"
    subprocess.run([cc, f"-I{ROOT / 'include'}", str(probe), "-o", str(exe)], check=True)
    sizes, offs = subprocess.run([str(exe)], capture_output=True, text=True,
                                 check=True).stdout.split("\n")[:2]
    expect = [C.sizeof(t) for t in (N.CylGridC, N.CartGridC, N.RayViewC, N.DetViewC,
                                    N.SamplingC, N.UpdateC, N.BatchC)]
    assert [int(x) for x in sizes.split()] == expect
    assert [int(x) for x in offs.split()] == [N.CylGridC.rot.offset, N.CylGridC.t.offset,
                                             N.UpdateC.weights.offset, N.BatchC.view_ids.offset,
                                             N.UpdateC.mu_peers.offset,
                                             N.UpdateC.n_peers.offset,
                                             N.UpdateC.peer_ranges.offset]


def test_argument_errors_return_status_not_crash():
    """Null pointers are rejected before any CUDA call (works without a GPU)."""
    from paper_2005_11976_b200 import _native as N
    lib = N.load_library()
    b = N.BatchC()
    s = N.SamplingC()
    g = N.CylGridC()
    rc = lib.ct_fp_cyl(None, None, C.byref(g), None, C.byref(b), C.byref(s), None, None, None)
    assert rc == -1
    assert lib.ct_last_error()
    with pytest.raises(N.NativeError):
        N.call("ct_sart_update", None, None, 0, 0, None, None)


def test_update_peer_lists_are_validated():
    """Every ct_update entry point rejects an inconsistent peer list before any
    launch (n_peers < 0, or n_peers > 0 without the pointer array), and the
    stand-alone update refuses peers (it writes mu only)."""
    from paper_2005_11976_b200 import _native as N
    lib = N.load_library()
    g = N.CylGridC(4, 8, 6, 0, 2.0, 3.0)
    gx = N.CartGridC(4, 4, 4, 0, 0.5)
    b = N.BatchC(1, 9, 9, 0, None)
    dummy = C.c_void_p(16)            # never dereferenced: validation comes first
    for n_peers, peers in ((-1, None), (2, None)):
        u = N.UpdateC(0.5, 1, None, dummy, peers, n_peers, 0)
        for rc in (lib.ct_bp_cyl_update(dummy, None, dummy, C.byref(b), C.byref(g), dummy,
                                        C.byref(u), None),
                   lib.ct_bp_cart_update(dummy, None, dummy, C.byref(b), C.byref(gx),
                                         C.byref(u), None),
                   lib.ct_bp_cyl_update_range(dummy, None, dummy, C.byref(b), C.byref(g), dummy,
                                              C.byref(u), 0, 1, None),
                   lib.ct_bp_cart_update_range(dummy, None, dummy, C.byref(b), C.byref(gx),
                                               C.byref(u), 0, 1, None),
                   lib.ct_sart_update(dummy, dummy, 0, 1, C.byref(u), None)):
            assert rc == -1
            assert b"peer" in lib.ct_last_error()
    u = N.UpdateC(0.5, 1, None, dummy, dummy, 1, 0)
    assert lib.ct_sart_update(dummy, dummy, 0, 1, C.byref(u), None) == -1


def test_gather_layout_query():
    """ct_gather_layout_*: the layout the FP of a config reads (no GPU needed)."""
    from paper_2005_11976_b200 import _native as N
    import paper_2005_11976_b200 as P
    from paper_2005_11976_b200 import _device as D
    lib = N.load_library()
    cyl = lambda *s: C.byref(D.grid_c(P.CylGrid(*s, 12.0, 24.0)))
    assert lib.ct_gather_layout_cyl(cyl(256, 512, 256)) == 1          # C2/C3: GL_OCT
    assert lib.ct_gather_layout_cyl(cyl(512, 1024, 384)) == 2         # C4-cyl/C5: GL_QUAD
    cart = D.grid_c(P.CartGrid.centered(512, 512, 512, 24.0 / 512))
    assert lib.ct_gather_layout_cart(C.byref(cart)) == 3              # C4-cart: GL_OCTB
    assert lib.ct_gather_layout_cyl(C.byref(N.CylGridC())) == -1


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_2005_11976_b200 as P
    from paper_2005_11976_b200.errors import NativeUnavailable
    g = P.CylGrid(4, 8, 6, 2.0, 3.0)
    geom = P.ScanGeometry(791.0, 679.0, 9, 9, 0.748, (4.0, 4.0), [0.0])
    with pytest.raises(NativeUnavailable):
        P.forward_project(P.CylVolume.zeros(g), geom, 0)
    with pytest.raises(NativeUnavailable):
        P.back_project(np.zeros((9, 9)), geom, 0, g)
    ps = P.ProjectionSet(geom, np.zeros((1, 9, 9)))
    with pytest.raises(NativeUnavailable):
        P.sart_run(ps, g, P.SartConfig())


def test_product_does_not_import_oracle():
    """The oracle is test infrastructure only: no product module references it."""
    pkg = ROOT / "paper_2005_11976_b200"
    for f in pkg.rglob("*.py"):
        src = f.read_text()
        assert "import oracle" not in src and "liboracle" not in src, f
    for f in pkg.rglob("*.cu"):
        src = f.read_text()
        assert "liboracle" not in src and not re.search(r"#include.*oracle", src), f
