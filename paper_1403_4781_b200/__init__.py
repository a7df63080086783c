"""sparsedict-B200: the split-and-merge dictionary-learning hot path of
arXiv 1403.4781 (reference package ``sparsedict``) on NVIDIA B200 (sm_100a).

Drop-in surface for the hot path (reference __init__.py:67-117): OMP coding,
MOD update and atom replacement, standard / local / merge / split-merge
training, denoising and mse_db. All arithmetic runs in libsdb200.so.
"""

__version__ = "0.1.0"

from ._engine import get_precision, set_precision
from .exceptions import FormatError, InvalidInputError, SparsedictError
from .sparse_coding import (
    OmpDiagnostics,
    SparseCodeMatrix,
    SparseVector,
    check_dictionary,
    omp_batch,
    omp_error_bound,
    omp_fixed_sparsity,
)
