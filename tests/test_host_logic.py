"""Host-side logic of the drop-in API (CPU only): validation raises
InvalidInputError before any launch, exactly where the reference does;
seeded split / seed derivation match the reference's golden vectors."""

import numpy as np
import pytest

import paper_1403_4781_b200 as sdb
from conftest import load_golden
from paper_1403_4781_b200.trainer import _derive_seeds

TRN = load_golden("train_golden.npz")


def test_split_indices_matches_reference():
    blocks = sdb.split_indices(103, 7, seed=11)
    assert np.array_equal(np.concatenate(blocks), TRN["split__idx"])
    assert [b.size for b in blocks] == list(TRN["split__sizes"])
    assert [b.size for b in sdb.split_indices(10, 3, seed=0)] == [4, 3, 3]


def test_derive_seeds_matches_reference():
    assert _derive_seeds(123, 9) == [int(v) for v in TRN["seeds"]]


def test_split_dataset_columns(rng):
    Y = rng.standard_normal((6, 23))
    for shard, ids in zip(sdb.split_dataset(Y, 4, seed=1), sdb.split_indices(23, 4, seed=1)):
        assert np.array_equal(shard, Y[:, ids])


def test_split_rejects_oversized_L():
    with pytest.raises(sdb.InvalidInputError):
        sdb.split_indices(5, 6, seed=0)


@pytest.mark.parametrize("kwargs", [
    dict(K=0, s=3), dict(K=20, s=0), dict(K=20, s=3, iterations=0), dict(K=20, s=3, init="bogus"),
    dict(K=20, s=3, mode="bogus"), dict(K=20, s=4, mode="split-merge", L=2),
    dict(K=20, s=4, mode="split-merge", L=2, K1=10, s1=3, s2=2),
    dict(K=20, s=4, mode="split-merge", L=2, K1=30, s1=2, s2=2),
    dict(K=20, s=3, eps=-1.0), dict(K=20, s=3, precision="fp16"),
])
def test_train_config_rejects_invalid(kwargs):
    with pytest.raises(sdb.InvalidInputError if "precision" not in kwargs else ValueError):
        sdb.TrainConfig(**kwargs).validate()


def test_train_config_round_trip():
    cfg = sdb.TrainConfig(K=20, s=4, iterations=7, seed=3, mode="split-merge", L=4, K1=10, s1=2,
                          s2=2)
    assert sdb.TrainConfig.from_dict(cfg.to_dict()) == cfg
    with pytest.raises(sdb.InvalidInputError):
        sdb.TrainConfig.from_dict({"K": 20, "s": 3, "bogus": 1})
    ext = sdb.TrainConfig(K=20, s=3, eps=1.5, s_max=6, precision="fp32")
    assert sdb.TrainConfig.from_dict(ext.to_dict()) == ext


def test_containers():
    x = sdb.SparseVector(6, np.array([1, 4]), np.array([2.0, -3.0]))
    assert x.nnz == 2 and np.array_equal(x.to_dense(), [0, 2.0, 0, 0, -3.0, 0])
    with pytest.raises(sdb.InvalidInputError):
        sdb.SparseVector(6, np.array([4, 1]), np.array([1.0, 1.0]))
    with pytest.raises(sdb.InvalidInputError):
        sdb.SparseVector(3, np.array([3]), np.array([1.0]))
    X = sdb.SparseCodeMatrix.from_columns(6, [x, sdb.SparseVector(6, np.array([0]), np.array([1.0]))])
    assert X.N == 2 and X.nnz == 3 and list(X.row_usage()) == [1, 1, 0, 0, 1, 0]
    assert X == sdb.SparseCodeMatrix(6, X.indptr, X.indices, X.data)


def test_validation_before_any_launch(rng):
    """Every precondition the reference checks raises on the host, so these
    run without a GPU."""
    D = rng.standard_normal((6, 9))
    D /= np.linalg.norm(D, axis=0)
    with pytest.raises(sdb.InvalidInputError):
        sdb.omp_fixed_sparsity(np.full(6, np.nan), D, 2)
    with pytest.raises(sdb.InvalidInputError):
        sdb.omp_fixed_sparsity(np.ones(6), D, 7)
    with pytest.raises(sdb.InvalidInputError):
        sdb.omp_fixed_sparsity(np.ones(6), rng.standard_normal((6, 9)), 2)
    with pytest.raises(sdb.InvalidInputError):
        sdb.omp_error_bound(np.ones(6), D, -1.0, 3)
    with pytest.raises(sdb.InvalidInputError):
        sdb.omp_batch(rng.standard_normal((5, 3)), D, s=2)
    with pytest.raises(sdb.InvalidInputError):
        sdb.omp_batch(rng.standard_normal((6, 3)), D, s=2, eps=0.5)
    with pytest.raises(sdb.InvalidInputError):
        sdb.omp_batch(rng.standard_normal((6, 3)), D)
    with pytest.raises(sdb.InvalidInputError):
        sdb.merge_dictionaries([], K=5, s2=1, merge_iterations=1, seed=0)
    with pytest.raises(sdb.InvalidInputError):
        sdb.train_standard(rng.standard_normal((8, 40)),
                           sdb.TrainConfig(K=10, s=2, iterations=1, mode="split-merge", L=2, K1=5,
                                           s1=2, s2=1))
    with pytest.raises(sdb.InvalidInputError):
        sdb.train_split_merge(rng.standard_normal((8, 40)), sdb.TrainConfig(K=10, s=2, iterations=1))
    with pytest.raises(sdb.InvalidInputError):
        sdb.DenoiseConfig(sigma=1.0, stride=9).validate()


def test_empty_batch_without_gpu(rng):
    D = rng.standard_normal((8, 12))
    D /= np.linalg.norm(D, axis=0)
    X = sdb.omp_batch(np.empty((8, 0)), D, s=2)
    assert X.N == 0 and X.nnz == 0


def test_overcomplete_dct_matches_reference():
    DN = load_golden("denoise_golden.npz")
    np.testing.assert_allclose(sdb.overcomplete_dct(8, 256), DN["dct8"], rtol=0, atol=1e-15)
    np.testing.assert_allclose(sdb.overcomplete_dct(4, 64), DN["dct4"], rtol=0, atol=1e-15)
    with pytest.raises(sdb.InvalidInputError):
        sdb.overcomplete_dct(8, 49)


@pytest.mark.parametrize("n,seed", [(0, 1), (1, 2), (2, 3), (10, 0), (103, 11), (65537, 9),
                                    (1_000_003, 1234), (2_040_200, 5)])
def test_native_permutation_bitwise_numpy(n, seed):
    """The native split permutation == numpy.random.default_rng(seed).permutation(n)
    (trainer.py:208-209)."""
    from paper_1403_4781_b200 import _lib
    assert np.array_equal(_lib.permutation(n, seed), np.random.default_rng(seed).permutation(n))


def _numpy_swap_targets(n, seed):
    """Fisher-Yates targets of Generator.permutation(n): numpy's masked
    rejection on buffered 32-bit halves of the PCG64 output (restated)."""
    bg = np.random.default_rng(seed).bit_generator
    buf = []

    def next32():
        if not buf:
            r = int(bg.random_raw())
            buf.extend([r >> 32, r & 0xFFFFFFFF])
        return buf.pop()

    js = []
    for i in range(n - 1, 0, -1):
        mask = i
        for sh in (1, 2, 4, 8, 16):
            mask |= mask >> sh
        while True:
            v = next32() & mask
            if v <= i:
                break
        js.append(v)
    return np.array(js, dtype=np.uint32)


@pytest.mark.parametrize("n", [2, 3, 4, 5, 9, 16, 17, 1000, 4097])
def test_native_swap_targets_match_numpy(n):
    from paper_1403_4781_b200 import _lib
    for seed in (0, 11):
        js = np.empty(n - 1, dtype=np.uint32)
        assert _lib.swap_targets(n, seed, js)
        ref = _numpy_swap_targets(n, seed)
        assert np.array_equal(js, ref)
        a = np.arange(n)
        for k, j in enumerate(js):
            i = n - 1 - k
            a[i], a[j] = a[j], a[i]
        assert np.array_equal(a, np.random.default_rng(seed).permutation(n))
