"""paper_2603_28475_b200 — B200-native batched PNCG-IPC tactile stepper (Tac2Real hot path).

The product is the C-ABI library libtac.so (include/tac.h, sources in csrc/);
``TacSim`` is its thin Python binding.
"""
from .tac import (EXPORTED, FLAG_CONVERGED, FLAG_INFEASIBLE, FLAG_LARGE_MOTION, FLAG_MAXITER, FLAG_NAN,
                  FLAG_OVERFLOW, FLAG_STAGNATION, LIB_PATH, NcclComm, TacError, TacSim, lib, nccl_unique_id)

__all__ = ["TacSim", "TacError", "NcclComm", "nccl_unique_id", "lib", "LIB_PATH", "EXPORTED", "FLAG_CONVERGED", "FLAG_MAXITER", "FLAG_NAN",
           "FLAG_INFEASIBLE", "FLAG_LARGE_MOTION", "FLAG_OVERFLOW", "FLAG_STAGNATION"]
