"""CPU oracle for the BTTB fast-forward-operator hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s CPU-baseline leg (and ``bench.py --impl reference``) may import
this package, and only as the checker / the reference arm -- never as the thing
measured or shipped.  The product path (``paper_1912_06976_b200``) never
imports it and fails loudly when its CUDA library is missing.
"""
from .bttb_oracle import *  # noqa: F401,F403
