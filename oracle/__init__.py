"""CPU oracle for the HFTA fused training step (arXiv 2102.02344).

*** TEST INFRASTRUCTURE. ***  Only `tests/`, `__graft_entry__.smoke()` and
`bench.py`'s `cpu_baseline` / `--impl reference` legs may import or execute
anything under `oracle/`.  The product path (`paper_2102_02344_b200`) never
imports it and has no CPU fallback.

What it computes: one training step of B models, each trained ALONE in a
Python loop with its own hyper-parameters (the paper's invariant that fused
model b equals model b trained alone: App. C Eq. 1-6
P:L1325-1366, App. D).  NumPy float64 throughout.

Modules:
  layers  -- serial operator definitions with hand-written backward
             (App. B rows)
  adam    -- serial Adam, PyTorch-1.6 form (reading R7)
  philox  -- Philox4x32-10 for the dropout mask (reading R14)
  models  -- cfg1 MLP, PointNet-cls/seg, DCGAN per-model steps and the
             fused-step oracle (a loop over b)

Parity pins: tests/test_oracle_*.py (finite differences, PyTorch-CPU-fp64
functional ops, closed forms, Random123 known answers, brute force, the
serial-equals-fused invariants).  Functions without an independent pin:
none known ("parity unpinned" would be stated here and in DESIGN.md).
"""
from . import layers, adam, philox, models  # noqa: F401
