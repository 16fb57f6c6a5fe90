"""Build a scratch harness that runs the REFERENCE's own hot-path test modules
through the drop-in (VERDICT r1 "next round" 2).

    python scripts/make_reftests.py        # in the build container only

Writes the git-ignored directory ``_reftests/`` (never committed; it carries
the reference's tests and, renamed, its package for the names the drop-in does
not provide):
  _reftests/_sketchpress_ref/   copy of /root/reference/pkg/src/sketchpress
  _reftests/sketchpress/        alias package: every hot-path name resolves to
                                paper_2105_01271_b200; names off the hot path
                                (theorem bounds, codec, archive, CLI, datagen)
                                fall through to _sketchpress_ref
  _reftests/tests/              copies of pkg/tests/{conftest, test_sketch,
                                test_kernels, test_svd, test_power, test_rowid,
                                test_snapshot_io, test_acceptance}.py
Run on the GPU box with  cd _reftests && python -m pytest tests -p no:cacheprovider
and delete the directory afterwards (scripts/run_reftests.sh does both).
"""
import shutil
from pathlib import Path

REF = Path("/root/reference/pkg")
ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "_reftests"
MODULES = ["sketch", "svd", "power", "rowid", "kernels", "snapshot_io", "errors", "analysis"]
TESTS = ["conftest", "test_sketch", "test_kernels", "test_svd", "test_power", "test_rowid",
         "test_snapshot_io", "test_acceptance"]

SHIM_INIT = '''"""Alias of the drop-in under the reference's package name (test harness)."""
import _sketchpress_ref as _ref
from paper_2105_01271_b200 import *  # noqa: F401,F403  the drop-in's names win
import paper_2105_01271_b200 as _ours

for _n in dir(_ref):
    if not _n.startswith("_") and not hasattr(_ours, _n):
        globals()[_n] = getattr(_ref, _n)          # off the hot path: the reference's own
'''

SHIM_MOD = '''"""sketchpress.{mod}: the drop-in's module, the reference's for the rest."""
import importlib as _il

_ref = _il.import_module("_sketchpress_ref.{mod}")
_ours = _il.import_module("paper_2105_01271_b200.{mod}")
from _sketchpress_ref.{mod} import *  # noqa: F401,F403
from paper_2105_01271_b200.{mod} import *  # noqa: F401,F403


def __getattr__(name):
    if hasattr(_ours, name):
        return getattr(_ours, name)
    return getattr(_ref, name)
'''


def main():
    if OUT.exists():
        shutil.rmtree(OUT)
    (OUT / "sketchpress").mkdir(parents=True)
    (OUT / "tests").mkdir()
    shutil.copytree(REF / "src" / "sketchpress", OUT / "_sketchpress_ref")
    (OUT / "sketchpress" / "__init__.py").write_text(SHIM_INIT)
    for mod in MODULES:
        (OUT / "sketchpress" / f"{mod}.py").write_text(SHIM_MOD.format(mod=mod))
    for extra in ("archive", "codec", "config", "datagen", "cli"):
        (OUT / "sketchpress" / f"{extra}.py").write_text(
            f"from _sketchpress_ref.{extra} import *  # noqa: F401,F403  (off the hot path)\n"
            f"from _sketchpress_ref import {extra} as _m\n\n\ndef __getattr__(name):\n    return getattr(_m, name)\n")
    for t in TESTS:
        shutil.copy(REF / "tests" / f"{t}.py", OUT / "tests" / f"{t}.py")
    (OUT / "conftest.py").write_text(
        "import sys\nfrom pathlib import Path\n"
        "sys.path.insert(0, str(Path(__file__).resolve().parent))\n"
        "sys.path.insert(0, str(Path(__file__).resolve().parent.parent))\n")
    print("wrote", OUT)


if __name__ == "__main__":
    main()
