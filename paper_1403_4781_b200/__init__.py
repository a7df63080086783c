"""sparsedict-B200: the split-and-merge dictionary-learning hot path of
arXiv 1403.4781 (reference package ``sparsedict``) on NVIDIA B200 (sm_100a).

Drop-in surface for the hot path (reference __init__.py:67-117): OMP coding,
MOD update and atom replacement, standard / local / merge / split-merge
training, the denoising pipeline and mse_db. All arithmetic runs in
libsdb200.so (hand-written CUDA for sm_100a behind a C ABI); there is no CPU
fallback. The sparse-model generators (synthesis) are included, with an
on-device variant, and the reference's file formats (storage: SDICT, SDATA,
PGM) and command line (cli: gen / train / denoise / eval). Out of scope
(DESIGN.md): the cost model and the bench sweep harness.
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
from .dictionary_update import (
    ReplacementReport,
    UpdateDiagnostics,
    mod_update,
    normalize_columns,
    replace_degenerate_atoms,
)
from .trainer import (
    TrainConfig,
    TrainReport,
    merge_dictionaries,
    split_dataset,
    split_indices,
    train_local,
    train_split_merge,
    train_standard,
)
from .denoising import (
    DenoiseConfig,
    GrayImage,
    add_gaussian_noise,
    denoise_image,
    extract_patches,
    overcomplete_dct,
    reconstruct_from_patches,
)
from .metrics import atom_recovery, mse_db, psnr
from .synthesis import gen_dictionary, gen_signals, gen_signals_device
from .storage import load_dictionary, load_dataset, load_pgm, save_dataset, save_dictionary, save_pgm

__all__ = [
    "get_precision", "set_precision",
    "FormatError", "InvalidInputError", "SparsedictError",
    "OmpDiagnostics", "SparseCodeMatrix", "SparseVector", "check_dictionary", "omp_batch",
    "omp_error_bound", "omp_fixed_sparsity",
    "ReplacementReport", "UpdateDiagnostics", "mod_update", "normalize_columns",
    "replace_degenerate_atoms",
    "TrainConfig", "TrainReport", "merge_dictionaries", "split_dataset", "split_indices",
    "train_local", "train_split_merge", "train_standard",
    "DenoiseConfig", "GrayImage", "add_gaussian_noise", "denoise_image", "extract_patches",
    "overcomplete_dct", "reconstruct_from_patches",
    "atom_recovery", "mse_db", "psnr",
    "gen_dictionary", "gen_signals", "gen_signals_device",
    "load_dictionary", "load_dataset", "load_pgm", "save_dataset", "save_dictionary", "save_pgm",
]
