"""B200-native engine for MeCeFO's degraded-node training step (arXiv 2510.16415).

Drop-in for the step and failure-handling path of the reference simulator
`faultsim` (pkg/src/faultsim). The module layout mirrors the reference
(model, approx, linalg, cluster, optim, harness) with the same function
names and argument order, operating on CUDA tensors through libmecefo.so.
"""

__version__ = "0.1.0"
