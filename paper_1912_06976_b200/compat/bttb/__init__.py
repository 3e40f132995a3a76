"""Import shim: ``import bttb`` resolves to the sm_100a drop-in.

Put ``paper_1912_06976_b200/compat`` first on ``sys.path``
and unchanged callers of the reference's hot-path API get the GPU operator.
Dense assembly, the benchmark harness, the CLI and stack persistence are not
part of the drop-in (SURVEY.md section 2 scope).
"""
import sys as _sys

from paper_1912_06976_b200 import *  # noqa: F401,F403
from paper_1912_06976_b200 import __all__, __version__  # noqa: F401
from paper_1912_06976_b200 import grid, harness, kernels, multiply, transform  # noqa: F401

for _name in ("grid", "harness", "kernels", "multiply", "transform"):
    _sys.modules[f"{__name__}.{_name}"] = _sys.modules[f"paper_1912_06976_b200.{_name}"]
