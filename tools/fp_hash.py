"""Hash of forward projections + one OS-SART pass on the C2 and C5 workloads
(bit-identity check between library builds: CT_LIBRARY=... python tools/fp_hash.py)."""
import hashlib
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2005_11976_b200 as P  # noqa: E402
from paper_2005_11976_b200 import workloads as W  # noqa: E402
from paper_2005_11976_b200.recon import SartRun  # noqa: E402


def h(t):
    return hashlib.sha256(t.detach().cpu().numpy().tobytes()).hexdigest()[:16]


for name, wl in (("c2", W.c2_medium(n_views=24)), ("c5", W.c5_object(0, n_views=12))):
    vol = P.CylVolume(wl.grid, torch.as_tensor(wl.mu, device="cuda"))
    ps = P.forward_project_all(vol, wl.geom)
    run = SartRun(ps, wl.grid, P.SartConfig(relaxation=0.3, n_iterations=2, n_subsets=4))
    out, rep = run.run()
    print(name, h(ps.images), h(out.mu), repr(rep.residuals))
