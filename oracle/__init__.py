"""fp64 CPU oracle for the TPLA decode hot path (arXiv 2508.15881).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product (``paper_2508_15881_b200``, ``libtpla.so``) never imports,
links or executes anything here, and this package imports nothing from the
product: the two share no code.  Only ``synth/`` (seeded inputs, no method
arithmetic) is common to both.

Everything is NumPy float64, written to be checked against PAPER.md by eye:
no blocking, fusion or reordering beyond what the cited equation states.

Modules
-------
numerics  RMS / RMSNorm, softmax, bf16 rounding, splitmix64
reparam   Sylvester Hadamard, PCA, alpha/mu constants
plan      (k, g) shard plan
mla       MLA: non-absorbed with decoupled RoPE (Eq. isolate_rope),
          absorbed (Eq. mla_softmax, absorption P:108-114)
tpla      TPLA: weight conversion, cache rows,
          per-device decode (Eq. tpla_softmax_one_device), all-reduce
cost      per-device KV widths and attention FLOPs

Parity status: every public function is pinned by ``tests/test_oracle_pins.py``
except where a docstring says "parity unpinned" (also listed in DESIGN.md).
"""
from . import numerics, reparam, plan, mla, tpla, cost  # noqa: F401
