"""Host-side mirror of the reference csr.py: generators (byte-identical for a
seed), EMGI IO, invariants, source picking."""
import os

import numpy as np
import pytest

from fixtures import crc, goldens

import paper_2006_06890_b200 as zc

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _check_graph(g, rec):
    assert g.num_vertices == rec["V"] and g.num_edges == rec["E"]
    assert crc(g.offsets, "<u8") == rec["offsets_crc_u8"]
    assert crc(g.edges, "<u4") == rec["edges_crc_u4"]
    if "weights_crc_u4" in rec:
        assert crc(g.weights, "<u4") == rec["weights_crc_u4"]


@pytest.mark.parametrize("key,args", [
    ("uniform_1000_16_48_s7", (1000, 16, 48, 7)),
    ("uniform_300_1_5_s9", (300, 1, 5, 9)),
    ("uniform_4096_0_9_s3", (4096, 0, 9, 3)),
    ("uniform_65536_16_16_s3", (65536, 16, 16, 3)),
])
def test_generate_uniform_matches_reference(key, args):
    g = zc.with_uniform_weights(zc.generate_uniform(args[0], args[1], args[2], seed=args[3]))
    _check_graph(g, goldens()["generator"][key])


@pytest.mark.parametrize("key,args", [
    ("powerlaw_100000_8.0_2.0_s3", (100000, 8.0, 2.0, 3)),
    ("powerlaw_3000_12.0_2.0_s1", (3000, 12.0, 2.0, 1)),
])
def test_generate_powerlaw_matches_reference(key, args):
    _check_graph(zc.generate_powerlaw(*args[:3], seed=args[3]), goldens()["generator"][key])


def test_symmetrized_matches_reference():
    g = zc.symmetrized(zc.generate_uniform(2 ** 10, 2, 6, seed=5))
    assert not g.directed
    _check_graph(g, goldens()["generator"]["sym_uniform_1024_2_6_s5"])


def test_pick_sources_matches_reference():
    g = zc.generate_uniform(1000, 16, 48, seed=7)
    assert zc.pick_sources(g, 4).tolist() == goldens()["pick_sources_1000_16_48_s7"]


def test_pick_sources_insufficient():
    g = zc.CsrGraph(3, 0, np.zeros(4, np.int64), np.zeros(0, np.int64))
    with pytest.raises(ValueError):
        zc.pick_sources(g, 1)


@pytest.mark.parametrize("eb,wb,weighted", [(4, 4, True), (8, 8, True), (4, 8, False)])
def test_emgi_roundtrip(tmp_path, eb, wb, weighted):
    g = zc.generate_uniform(500, 0, 9, seed=3, edge_elem_bytes=eb)
    if weighted:
        g = zc.with_uniform_weights(g, weight_elem_bytes=wb)
    p = str(tmp_path / "g.emgi")
    zc.store_csr_binary(g, p)
    with open(p, "rb") as fh:
        raw = fh.read()
    assert raw[:4] == b"EMGI"
    edge_off = -(-(28 + 8 * 501) // 128) * 128
    assert edge_off % 128 == 0
    h = zc.load_csr_binary(p)
    assert h == g
    assert h.edges.dtype.itemsize == eb  # kept at on-disk width
    assert zc.load_csr_binary(p, widen=True).edges.dtype == np.int64


def test_emgi_errors(tmp_path):
    p = str(tmp_path / "bad.emgi")
    with open(p, "wb") as fh:
        fh.write(b"XXXX" + bytes(40))
    with pytest.raises(ValueError, match="magic"):
        zc.load_csr_binary(p)
    g = zc.generate_uniform(100, 1, 3, seed=1)
    zc.store_csr_binary(g, p)
    with open(p, "rb") as fh:
        raw = fh.read()
    with open(p, "wb") as fh:
        fh.write(raw[:-5])
    with pytest.raises(ValueError, match="truncated"):
        zc.load_csr_binary(p)


def test_validate_rejects():
    ok = zc.generate_uniform(50, 1, 3, seed=1)
    zc.validate(ok)
    bad = zc.CsrGraph(3, 2, np.array([0, 2, 1, 2]), np.array([1, 2]))
    with pytest.raises(ValueError, match="non-decreasing"):
        zc.validate(bad)
    bad = zc.CsrGraph(2, 1, np.array([0, 1, 1]), np.array([5]))
    with pytest.raises(ValueError, match="out of range"):
        zc.validate(bad)


def _reference():
    import oracle
    try:
        return oracle.reference()
    except ImportError:
        pytest.skip("reference package unavailable (no /root/reference, no oracle/_ref zip)")


def test_reference_csrgraph_duck_typing():
    """Graphs built by the reference itself are accepted (duck typing)."""
    ref = _reference()
    g = ref.generate_uniform(200, 1, 5, seed=2)
    assert zc.pick_sources(g, 2).tolist() == ref.pick_sources(g, 2).tolist()
    zc.validate(g)


def test_load_edge_list_text_matches_reference_fixture(tmp_path):
    """load_edge_list_text against the reference's own outputs
    (tests/golden/make_golden_text.py; csr.py:123-177): CSR arrays, vertex
    count, weights, and the ValueError messages."""
    import json
    rows = json.loads(str(np.load(os.path.join(GOLDEN, "edge_list_text.npz"))["cases"]))
    assert len(rows) >= 100
    for k, row in enumerate(rows):
        path = tmp_path / f"case{k}.txt"
        path.write_text(row["text"])
        if "error" in row:
            with pytest.raises(ValueError) as exc:
                zc.load_edge_list_text(str(path), directed=row["directed"],
                                       num_vertices=row["num_vertices"])
            assert str(exc.value) == row["error"], k
            continue
        g = zc.load_edge_list_text(str(path), directed=row["directed"],
                                   num_vertices=row["num_vertices"])
        assert g.num_vertices == row["nv_out"] and g.directed == row["directed"], k
        assert g.offsets.tolist() == row["offsets"] and g.edges.tolist() == row["edges"], k
        assert (None if g.weights is None else g.weights.tolist()) == row["weights"], k
