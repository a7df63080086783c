"""Host -> device ingestion of ordinary (pageable) numpy arrays: the threaded
staging ring (upload_pageable) must deliver exactly the source bytes, for both
memory orders, for sizes around the chunk boundaries, and back to back."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("order", ["C", "F"])
def test_upload_pageable_is_exact(order):
    from paper_1403_4781_b200 import _engine as E
    rng = np.random.default_rng(5)
    ch = E.UPLOAD_CHUNK
    for n_cols in (3, (2 * ch) // 64 + 1, (3 * ch) // 64 + 17):     # small copy, 2+ and 3+ chunks
        Y = np.asarray(rng.standard_normal((64, n_cols)), order=order)
        for _ in range(2):                                        # the ring is reused across calls
            T = E.upload_pageable(Y)
            assert tuple(T.shape) == Y.shape
            assert np.array_equal(T.cpu().numpy(), Y)
        Y[:, -1] += 1.0                                            # a later call must see new contents
        assert np.array_equal(E.upload_pageable(Y).cpu().numpy(), Y)


def test_ingest_matches_plain_copy():
    import torch
    from paper_1403_4781_b200 import _engine as E
    rng = np.random.default_rng(6)
    Y = rng.standard_normal((64, 300000))                          # > 2 chunks (C order, m x N)
    Yd, bad = E.ingest_signals(Y, "fp32")
    assert int(bad.item()) == 0
    ref = torch.from_numpy(np.ascontiguousarray(Y.T)).to(E.device()).float()
    assert torch.equal(Yd, ref)
