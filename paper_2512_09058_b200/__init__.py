"""B200-native (sm_100a) KKT factor+solve for linear-quadratic optimal
control problems -- the linear-solver hot path of arXiv 2512.09058
("Cyqlone"): per-partition Riccati recursion, Schur condensation, cyclic
reduction and substitution as FP64 DMMA CUDA kernels behind a C ABI
(include/cyqlone_b200.h). See DESIGN.md."""
from .ocp import EqOCPBatch, EqRhsBatch, EqSolutionBatch  # noqa: F401

__all__ = ["EqOCPBatch", "EqRhsBatch", "EqSolutionBatch"]
