"""Static check: no function reads a global its module never defines
(tools/lint_names.py -- the NameError-on-an-error-branch class of bug)."""

import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def test_no_undefined_globals():
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "lint_names.py")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stdout
