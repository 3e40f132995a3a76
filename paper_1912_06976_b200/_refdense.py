"""Dense assembly from the UNMODIFIED reference install (out of scope for the drop-in).

The dense sensitivity matrix (``/root/reference/pkg/src/bttb/dense.py``) is the
reference's O(m*n) oracle path; SURVEY.md section 8(b) keeps it coming from the
reference copy in ``baseline/_ref`` (``tools/install_reference.sh``) instead of
re-implementing it.  :func:`load` imports that file as
``paper_1912_06976_b200.dense``, so its relative imports (``.grid``,
``.kernels``) bind to this package: the dense matrices hold the same entries
as the device spectrum cache (the reference's own design -- dense and
transform paths share the entry generator, which its bit-exact layout tests
rely on, e.g. pkg/tests/test_transform.py:98-105).

Used by the benchmark harness (dense rows of the CSV, harness.py:88-168) and
by the ``bttb`` import shim.  Nothing on the operator's hot path imports it.
"""
import importlib.util
import os
import sys

_REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_NAME = __name__.rsplit(".", 1)[0] + ".dense"


def reference_install():
    """Directory holding the reference's ``bttb`` package (baseline/_ref by default)."""
    return os.environ.get("BTTB_REFERENCE_INSTALL", os.path.join(_REPO, "baseline", "_ref"))


def available():
    return os.path.isfile(os.path.join(reference_install(), "bttb", "dense.py"))


def load():
    """The reference dense module bound to this package; ModuleNotFoundError if absent."""
    if _NAME in sys.modules:
        return sys.modules[_NAME]
    path = os.path.join(reference_install(), "bttb", "dense.py")
    if not os.path.isfile(path):
        raise ModuleNotFoundError(
            f"dense assembly comes from the reference install, missing at {reference_install()} "
            "(run tools/install_reference.sh)")
    spec = importlib.util.spec_from_file_location(_NAME, path)
    mod = importlib.util.module_from_spec(spec)
    sys.modules[_NAME] = mod
    try:
        spec.loader.exec_module(mod)
    except Exception:
        del sys.modules[_NAME]
        raise
    return mod
