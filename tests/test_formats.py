"""File formats on the host: the "PKKV" KV dump written
and read by the package (paper_2512_24449_b200.tensor_model) against the
oracle's restatement, and the oracle's "PKKS" store file round trip."""
import numpy as np
import pytest

from oracle import packkv_oracle as O
from paper_2512_24449_b200 import errors as E
from paper_2512_24449_b200 import tensor_model as TM


@pytest.mark.parametrize("T", [0, 1, 37])
def test_dump_round_trip_and_matches_oracle(tmp_path, T):
    rng = np.random.default_rng(T)
    k = rng.standard_normal((2, 3, T, 16)).astype(np.float16)
    v = rng.standard_normal((2, 3, T, 16)).astype(np.float16)
    TM.write_dump(k, v, tmp_path / "a.pkkv")
    O.write_dump(k, v, tmp_path / "b.pkkv")
    assert (tmp_path / "a.pkkv").read_bytes() == (tmp_path / "b.pkkv").read_bytes()
    k2, v2 = TM.read_dump(tmp_path / "b.pkkv")
    assert k2.view(np.uint16).tobytes() == k.view(np.uint16).tobytes()
    assert v2.view(np.uint16).tobytes() == v.view(np.uint16).tobytes()
    k3, v3 = O.read_dump(tmp_path / "a.pkkv")
    assert np.array_equal(k3.view(np.uint16), k.view(np.uint16))
    assert (tmp_path / "a.pkkv").stat().st_size == 16 + 2 * 2 * 2 * 3 * T * 16


def test_dump_errors(tmp_path):
    k = np.ones((1, 1, 4, 8), np.float16)
    TM.write_dump(k, k, tmp_path / "a")
    data = (tmp_path / "a").read_bytes()
    cases = [(b"PKKX" + data[4:], E.BadMagicError), (data[:-1], E.TruncatedDumpError), (data[:10], E.TruncatedDumpError)]
    bad = bytearray(data)
    bad[16:18] = np.array([np.inf], np.float16).tobytes()
    cases.append((bytes(bad), E.NonFiniteValueError))
    for blob, err in cases:
        (tmp_path / "b").write_bytes(blob)
        with pytest.raises(err):
            TM.read_dump(tmp_path / "b")
        with pytest.raises(err):
            O.read_dump(tmp_path / "b")
    with pytest.raises(E.NonFiniteValueError):
        TM.write_dump(np.full((1, 1, 1, 2), np.nan, np.float16), k[:, :, :1, :2], tmp_path / "c")


def test_oracle_pkks_round_trip(tmp_path):
    rng = np.random.default_rng(5)
    H, D = 2, 64
    st = O.OracleStore(1, H, D, repack="v_median")
    st.compress_batch(0, rng.standard_normal((150, H, D)).astype(np.float16),
                      rng.standard_normal((150, H, D)).astype(np.float16))
    O.save_pkks(st, tmp_path / "s")
    back = O.load_pkks(tmp_path / "s")
    assert back.layer_stream(0) == st.layer_stream(0)
    assert np.array_equal(back.stage_k[0], st.stage_k[0])
    O.save_pkks(back, tmp_path / "t")
    assert (tmp_path / "s").read_bytes() == (tmp_path / "t").read_bytes()
    with pytest.raises(E.StoreFormatError):
        (tmp_path / "u").write_bytes((tmp_path / "s").read_bytes()[:-1])
        O.load_pkks(tmp_path / "u")


def test_repacker_cost_model_host():
    """The SPEC cost model (host arithmetic) against the oracle's."""
    from paper_2512_24449_b200 import repacker as R
    rng = np.random.default_rng(3)
    for _ in range(20):
        g = rng.integers(0, 1000, (int(rng.integers(1, 17)), int(rng.integers(1, 40))))
        assert R.pack_cost(g) == O.pack_cost(g)
    X = rng.integers(0, 50, (30, 7))
    perm = rng.permutation(30)
    assert R.plan_cost(X, perm, 8) == O.plan_cost(X, perm, 8)
    assert R.pack_cost(np.array([[0, 5], [3, 1]])) == 50
