"""Per-frame export wire format (a-13) vs bytes the reference produced
(tests/golden/codec.npz).  CPU only."""

import numpy as np
import pytest

from conftest import load_golden


@pytest.fixture(scope="module")
def C():
    from paper_2409_07759_b200 import codec
    return codec


def _arr(d):
    import paper_2409_07759_b200 as P
    return P.GaussianArrays(d["means"], d["quats"], d["scales"], d["opacities"], d["colors"])


@pytest.mark.parametrize("pid", [0, 1])
def test_records_and_slices_byte_identical(C, pid):
    import paper_2409_07759_b200 as P
    d = load_golden("codec")
    arr = _arr(d)
    prof = C.PROFILES[pid]
    assert C.encode_records(arr, prof) == d[f"records_p{pid}"].tobytes()
    assert C.pack_slice(arr, P.Lifespan(7, 7, 12), prof, swin_size=5) == d[f"slice_p{pid}"].tobytes()
    dec = C.decode_records(d[f"records_p{pid}"].tobytes(), prof)
    np.testing.assert_array_equal(dec.rows(), d[f"decoded_p{pid}"])


def test_quantized_record_is_30_bytes_and_byte_stable(C):
    d = load_golden("codec")
    prof = C.PROFILES[1]
    raw = d["records_p1"].tobytes()
    assert len(raw) == 30 * len(d["opacities"])
    again = C.encode_records(C.decode_records(raw, prof), prof)
    assert again == raw


def test_container_bytes(C, tmp_path):
    import paper_2409_07759_b200 as P
    d = load_golden("codec")
    arr = _arr(d).take(np.arange(10))
    man = C.Manifest(num_gs=20, swin_size=2, fps=30.0, total_frames=3, profile_id=1,
                     scene_bounds=(-1, -1, -1, 1, 1, 1), camera_count=2)
    with C.ContainerWriter(tmp_path / "c.swin", man) as w:
        for i, birth in enumerate([0, 0, 1, 2, 3]):
            w.write_slice(C.pack_slice(arr, P.Lifespan(birth, birth, birth + 2), C.PROFILES[1],
                                       swin_size=2, slice_index=(i if i < 2 else None)))
    assert (tmp_path / "c.swin").read_bytes() == d["container"].tobytes()
    with C.ContainerReader(tmp_path / "c.swin") as r:
        assert r.complete and r.num_sections == 5
        assert r.slice_targets == [1, 2, 3]
        gens = r.all_generations()
        assert [g.lifespan.expire for g in gens[:2]] == [2, 1]


def test_corruption_detected(C, tmp_path):
    d = load_golden("codec")
    raw = bytearray(d["container"].tobytes())
    raw[60] ^= 0xFF
    (tmp_path / "bad.swin").write_bytes(bytes(raw))
    with C.ContainerReader(tmp_path / "bad.swin") as r:
        with pytest.raises(C.CodecError):
            r.genesis_bytes()


def test_bandwidth_budget(C):
    import paper_2409_07759_b200 as P
    sp = P.StreamParams(swin_size=5, num_gs=200_000, fps=30.0, bytes_per_gaussian=30,
                        total_frames=300)
    bw = C.bandwidth(sp)
    assert bw.payload_bytes_per_s == 30 * 40_000 * 30.0
    assert 40_000 * 30 + C.HEADER_SIZE == 1_200_016
