"""ORACLE — TEST INFRASTRUCTURE ONLY. NOT PART OF THE PRODUCT.

A float64 numpy restatement of the reference's MeCeFO step path
(pkg/src/faultsim, arXiv 2510.16415) used as the checker for the CUDA
engine. Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s CPU
baseline leg (`cpu_baseline` / `--impl reference`) may import it.

Pinning: every function here is checked against golden vectors produced by
running the reference itself in the build container
(tests/golden/make_golden.py -> tests/golden/*.npz / *.json); see
tests/test_oracle_golden.py.

Modules
  model_ref    model.py / approx.py / linalg.py math (forward, exact and
               neighbor backward, low-rank Wgrad, CE, subspace iteration)
  cluster_ref  cluster.py control plane (NDB takeover, injection, active
               sets, Eq. (1) aggregation)
  optim_ref    optim.py AdamW / apply_step / lr schedule
"""
