"""File formats shared with the reference (io.cpp):
TSPW weights and TuneResult / DataflowConfig JSON, checked against the
compiled reference's own reader/writer (test_net_io.cpp cases) -- files move
between the CPU reference and sk200 unchanged."""
import os

import numpy as np
import pytest


@pytest.fixture(scope="module")
def io():
    from paper_2311_12862_b200 import io
    return io


@pytest.fixture(scope="module")
def ref_io(reference):
    if not reference.has_io:
        pytest.skip("reference built without io.cpp (no json.hpp)")
    return reference


def weights(seed=9):
    rng = np.random.default_rng(seed)
    shapes = [(27, 4, 16), (27, 16, 16), (8, 16, 32), (1, 32, 32), (27, 32, 16)]
    return [rng.standard_normal(s).astype(np.float32) for s in shapes]


def test_tspw_roundtrip_byte_identical(io, tmp_path):  # test_net_io.cpp:247-260
    p1, p2 = str(tmp_path / "w.tspw"), str(tmp_path / "w2.tspw")
    w = weights()
    io.write_tspw(p1, w)
    rd = io.read_tspw(p1)
    assert [a.shape for a in rd] == [a.shape for a in w]
    assert all(np.array_equal(a, b) for a, b in zip(rd, w))
    io.write_tspw(p2, rd)
    assert open(p1, "rb").read() == open(p2, "rb").read()


def test_tspw_corrupt_files(io, tmp_path):  # test_net_io.cpp:262-270
    from paper_2311_12862_b200.sparse import ValidationError
    p = str(tmp_path / "bad.tspw")
    for content in (b"TSPWxxxx", b"NOPE", b"TSPW" + (2).to_bytes(4, "little") + bytes(4)):
        open(p, "wb").write(content)
        with pytest.raises(ValidationError):
            io.read_tspw(p)
    io.write_tspw(p, weights()[:1])
    open(p, "ab").write(b"\0")
    with pytest.raises(ValidationError):
        io.read_tspw(p)


def test_tspw_interchange_with_reference(io, ref_io, tmp_path):
    w = weights(3)
    p_ours, p_ref = str(tmp_path / "ours.tspw"), str(tmp_path / "ref.tspw")
    io.write_tspw(p_ours, w)
    back = ref_io.tspw_read(p_ours)  # the reference reads our file
    assert all(np.array_equal(a.astype(np.float32), b) for a, b in zip(back, w))
    ref_io.tspw_write(p_ref, [a.astype(np.float64) for a in w])  # and we read its file
    assert open(p_ours, "rb").read() == open(p_ref, "rb").read()
    assert all(np.array_equal(a, b) for a, b in zip(io.read_tspw(p_ref), w))


def test_tune_result_matches_reference_json(io, ref_io):  # test_net_io.cpp:285-314
    from paper_2311_12862_b200 import sparse as sk
    text = ref_io.tune_sample()
    res = io.tune_result_from_json(text)
    assert io.tune_result_to_json(res) == text  # byte-identical to nlohmann dump(2)
    g = res.groups[0]
    assert g.forward == sk.DataflowConfig(sk.IMPLICIT_GEMM, 3, sk.tile_large())
    assert g.dgrad == sk.DataflowConfig(sk.FETCH_ON_DEMAND)
    assert g.wgrad is None and res.seed == 42 and res.log[0][3] == 3.25
    f, d, w = res.assignment()[0]
    assert d == g.dgrad and w == g.forward  # wgrad falls back to forward
    # a result written here is read back identically by the reference
    ours = io.tune_result_to_json(res)
    assert ref_io.tune_roundtrip(ours) == ours


def test_dataflow_config_json(io):
    from paper_2311_12862_b200 import sparse as sk
    from paper_2311_12862_b200.sparse import ValidationError
    for cfg in [sk.DataflowConfig(sk.GATHER_GEMM_SCATTER), sk.DataflowConfig(sk.FETCH_ON_DEMAND),
                sk.DataflowConfig(sk.IMPLICIT_GEMM, 2, sk.tile_small()),
                sk.DataflowConfig(sk.IMPLICIT_GEMM, 4, sk.tile_large(), 1)]:
        assert io.dataflow_config_from_json(io.dataflow_config_to_json(cfg)) == cfg
    for bad in ['{not json', '{"kind": "magic"}', '{"kind": "implicit_gemm", "reorder": "x"}']:
        with pytest.raises(ValidationError):
            io.dataflow_config_from_json(bad)
