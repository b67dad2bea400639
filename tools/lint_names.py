"""Report names that a function reads as globals but the module never defines.

    python tools/lint_names.py [files...]      (default: the package, bench.py,
                                                __graft_entry__.py, tools/, oracle/)

No linter ships in the image; this catches the NameError class of bug
(a missing import on a rarely-taken error branch) with the stdlib symtable.
"""

from __future__ import annotations

import builtins
import sys
import symtable
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def module_names(top: symtable.SymbolTable) -> set:
    return {s.get_name() for s in top.get_symbols()
            if s.is_assigned() or s.is_imported() or s.is_namespace()}


def walk(table, defined, path, out):
    for sym in table.get_symbols():
        if (sym.is_referenced() and (sym.is_global() or sym.is_declared_global())
                and sym.get_name() not in defined and not hasattr(builtins, sym.get_name())
                and sym.get_name() not in ("__file__", "__name__", "__doc__", "__spec__")):
            out.append(f"{path}: {table.get_name()}: undefined global {sym.get_name()!r}")
    for child in table.get_children():
        walk(child, defined, path, out)


def check(path: Path) -> list:
    src = path.read_text()
    top = symtable.symtable(src, str(path), "exec")
    defined = module_names(top)
    if "__all__" in src and "import *" in src:
        return []
    out = []
    for child in top.get_children():
        walk(child, defined, path.relative_to(ROOT), out)
    for sym in top.get_symbols():      # module-level reads
        if (sym.is_referenced() and not (sym.is_assigned() or sym.is_imported())
                and not hasattr(builtins, sym.get_name())
                and sym.get_name() not in ("__file__", "__name__", "__doc__", "__spec__")):
            out.append(f"{path.relative_to(ROOT)}: <module>: undefined {sym.get_name()!r}")
    return out


def main(argv):
    files = [Path(a).resolve() for a in argv] or sorted(
        [*ROOT.glob("paper_2005_11976_b200/*.py"), ROOT / "bench.py", ROOT / "__graft_entry__.py",
         *ROOT.glob("tools/*.py"), *ROOT.glob("oracle/*.py"), *ROOT.glob("tests/*.py")])
    problems = [p for f in files for p in check(f)]
    print("\n".join(problems) if problems else f"ok ({len(files)} files)")
    return 1 if problems else 0


if __name__ == "__main__":
    sys.exit(main(sys.argv[1:]))
