"""§8(f)-4 ABR tail-drop selection on the GPU (paper_2409_07759_b200.abr,
csrc/abr.cu) against the reference's own outputs (tests/golden/abr.npz, made
by tests/golden/make_golden.py from server.py:39-79) and, on large inputs, the
oracle's restatement.  Selection is index work: bit-exact."""

import math

import numpy as np
import pytest

from conftest import load_golden
from oracle import splat_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def A():
    from paper_2409_07759_b200 import abr
    return abr


def test_keep_indices_match_reference(A):
    d = load_golden("abr")
    for i, q in enumerate(d["fractions"]):
        assert np.array_equal(A.abr_keep_indices(d["opac"], float(q)), d[f"keep_{i}"])


def test_slice_bytes_match_reference(A):
    from paper_2409_07759_b200 import codec
    d = load_golden("abr")
    for pid in (0, 1):
        blob = d[f"slice_p{pid}"].tobytes()
        for i, q in enumerate(d["fractions"]):
            got = A.subsample_slice_bytes(blob, float(q), codec.PROFILES[pid])
            assert got == d[f"sub_p{pid}_{i}"].tobytes(), (pid, q)


@pytest.mark.parametrize("n", [1, 33, 1025, 200_003])
def test_large_and_ragged_with_ties_vs_oracle(A, n):
    rng = np.random.default_rng(n)
    op = rng.uniform(0, 1, n)
    op[rng.random(n) < 0.3] = 0.5            # one big tie class
    op[rng.random(n) < 0.05] = 0.0
    op[rng.random(n) < 0.02] = -0.0          # numpy ties -0.0 with 0.0
    op[:: max(n // 7, 1)] = 1.0
    for q in (1e-6, 0.01, 0.3, 0.5, 0.9, 0.999999, 1.0):
        got = A.abr_keep_indices(op, q)
        ref = O.abr_keep_indices(op, q)
        assert np.array_equal(got, ref), (n, q)
        assert len(got) == min(n, math.ceil(q * n))


def test_u8_profile_records_vs_oracle(A):
    """Profile-1 wire records (u8 opacity: 256 tie classes) at 50k records."""
    from paper_2409_07759_b200 import codec
    from paper_2409_07759_b200.core import GaussianArrays, Lifespan
    rng = np.random.default_rng(7)
    n = 50_000
    q = rng.normal(size=(n, 4))
    arr = GaussianArrays(rng.uniform(-1, 1, (n, 3)), q / np.linalg.norm(q, axis=1, keepdims=True),
                         np.exp(rng.uniform(-5, -1, (n, 3))), rng.uniform(0, 1, n),
                         rng.uniform(0, 1, (n, 3)))
    for pid in (0, 1):
        prof = codec.PROFILES[pid]
        blob = codec.pack_slice(arr, Lifespan(3, 3, 8), prof, 5)
        for f in (0.05, 0.5, 0.93):
            got = A.subsample_slice_bytes(blob, f, prof)
            body, kept = O.subsample_records(blob[O.SLICE_HEADER:], pid, f)
            assert got[O.SLICE_HEADER:] == body
            assert codec.SliceHeader.from_bytes(got).kept_count == kept


def test_subsample_arrays_and_errors(A):
    from paper_2409_07759_b200.core import GaussianArrays, InvalidParameterError
    rng = np.random.default_rng(3)
    n = 40
    q = rng.normal(size=(n, 4))
    arr = GaussianArrays(rng.uniform(-1, 1, (n, 3)), q / np.linalg.norm(q, axis=1, keepdims=True),
                         np.full((n, 3), 0.1), rng.uniform(0, 1, n), rng.uniform(0, 1, (n, 3)))
    kept, k = A.abr_subsample(arr, 0.4)
    assert k == 16 and len(kept) == 16
    assert np.array_equal(kept.opacities, arr.opacities[O.abr_keep_indices(arr.opacities, 0.4)])
    kept, k = A.abr_subsample(arr, 1.0)
    assert k == n
    for bad in (0.0, -0.1, 1.5):
        with pytest.raises(InvalidParameterError):
            A.abr_keep_indices(np.array([0.5]), bad)
    assert len(A.abr_keep_indices(np.zeros(0), 0.5)) == 0
