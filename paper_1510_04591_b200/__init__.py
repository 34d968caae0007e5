"""hsseig_b200: B200-native (sm_100a) divide-and-conquer merge step of arXiv 1510.04591.

Mirror of the reference package ``hsseig``'s merge-path API; compute runs in
libhsseig_b200.so (hand-written CUDA, FP64 DMMA), PyTorch only owns buffers.
"""
from .cauchy import CauchyEvecMatrix
from .dc import (EigenResult, MergeRecord, SolverConfig, merge_update, srrsc_cap,
                 update_vectors_dense, update_vectors_hss)
from .flops import FlopCounter
from .hss import (HssPartition, HssTree, build_partition, estimate_rank, hss_matmul_right,
                  hss_to_dense, interpolative_decomp, rand_hss_construct, rank_bound,
                  srrsc_hss_construct)
from .matgen import (FAMILIES, SymTridiagonal, gen_clement, gen_config5, gen_hermite, gen_kac,
                     gen_laguerre, gen_legendre, gen_toeplitz, gen_uniform, isolated_merge_system)
from .solver import adc_solve
from .secular import (RankOneSystem, SecularConvergenceError, SecularSolution,
                      WeightRecomputationError, column_normalizers, recompute_weights,
                      solve_secular)

BACKEND = "b200"
__version__ = "0.1.0"
