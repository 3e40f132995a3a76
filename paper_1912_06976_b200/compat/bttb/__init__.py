"""Import shim: ``import bttb`` resolves to the sm_100a drop-in.

Put ``paper_1912_06976_b200/compat`` first on ``sys.path`` (INTEGRATION.md
section 1) and unchanged callers of the reference API get the GPU operator:
the hot path (kernel entries, spectrum cache, forward / transpose products),
the persistence, the harness and the CLI all come from the drop-in.

The reference's public names are all exported (/root/reference/pkg/src/bttb/
__init__.py:9-31).  Dense assembly is out of scope for the drop-in (SURVEY.md
section 8(b)): ``assemble_dense``, ``dense_apply``, ``DenseSensitivity``,
``MemoryGuardError``, ``dump_layer_csv`` and ``DEFAULT_MEM_GUARD_BYTES`` are
the UNMODIFIED reference dense module from ``baseline/_ref``
(``tools/install_reference.sh``; override with ``BTTB_REFERENCE_INSTALL``),
loaded by ``paper_1912_06976_b200._refdense`` with its relative imports bound
to the drop-in -- so, as in the reference, the dense matrices and the
transform path share one entry generator (the reference's bit-exact layout
tests rely on that, pkg/tests/test_transform.py:98-105).  The entries
themselves are pinned against the reference's numpy entries by this repo's
own tests (tests/test_gpu_entries.py).
"""
import sys as _sys

from paper_1912_06976_b200 import *  # noqa: F401,F403
from paper_1912_06976_b200 import __all__ as _dropin_all
from paper_1912_06976_b200 import __version__  # noqa: F401
from paper_1912_06976_b200 import _refdense, cli, grid, harness, kernels, multiply, transform  # noqa: F401

for _name in ("cli", "grid", "harness", "kernels", "multiply", "transform"):
    _sys.modules[f"{__name__}.{_name}"] = _sys.modules[f"paper_1912_06976_b200.{_name}"]

_DENSE_NAMES = ("DEFAULT_MEM_GUARD_BYTES", "DenseSensitivity", "MemoryGuardError", "assemble_dense",
                "dense_apply", "dump_layer_csv")

if _refdense.available():
    dense = _refdense.load()
    _sys.modules[f"{__name__}.dense"] = dense
    DEFAULT_MEM_GUARD_BYTES = dense.DEFAULT_MEM_GUARD_BYTES
    DenseSensitivity = dense.DenseSensitivity
    MemoryGuardError = dense.MemoryGuardError
    assemble_dense = dense.assemble_dense
    dense_apply = dense.dense_apply
    dump_layer_csv = dense.dump_layer_csv
else:
    _MISSING = ("dense assembly comes from the reference install, which is missing at "
                f"{_refdense.reference_install()} (run tools/install_reference.sh)")
    from paper_1912_06976_b200.harness import DEFAULT_MEM_GUARD_BYTES  # noqa: F401

    class MemoryGuardError(RuntimeError):
        pass

    class DenseSensitivity:  # noqa: D101
        def __init__(self, *a, **k):
            raise ModuleNotFoundError(_MISSING)

    def _missing(*a, **k):
        raise ModuleNotFoundError(_MISSING)

    assemble_dense = dense_apply = dump_layer_csv = _missing

__all__ = sorted(set(_dropin_all) | set(_DENSE_NAMES))
