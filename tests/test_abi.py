"""The C-ABI library loads and exports every symbol include/zcgraph.h declares;
host-side argument checks raise the reference's ValueErrors without a GPU."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2006_06890_b200 as zc
from paper_2006_06890_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "zcgraph.h")
PROBE_HEADER = os.path.join(ROOT, "include", "zcprobe.h")


def header_functions(path=HEADER):
    text = open(path).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(zc_\w+)\s*\(", text, re.M)))


def exported_symbols(path):
    out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True,
                         text=True, check=True).stdout
    return set(re.findall(r" T (zc_\w+)", out))


def test_header_declares_expected_api():
    fns = header_functions()
    for name in ("zc_graph_create", "zc_graph_destroy", "zc_bfs", "zc_sssp", "zc_cc",
                 "zc_last_error", "zc_run_log"):
        assert name in fns
    assert set(fns) == set(_native.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = _native.lib()
    exported = exported_symbols(_native.LIB_PATH)
    missing = set(header_functions()) - exported
    assert not missing, missing
    # the product ABI is exactly the header: no probe / debug entry points
    assert exported == set(header_functions()), exported - set(header_functions())
    for name in header_functions():
        assert hasattr(lib, name)


def test_probe_library_is_separate():
    probes = header_functions(PROBE_HEADER)
    assert set(probes) == set(_native.PROBE_EXPORTED)
    assert not set(probes) & set(header_functions())
    assert set(probes) <= exported_symbols(_native.PROBE_LIB_PATH)
    lib = _native.probe_lib()
    for name in probes:
        assert hasattr(lib, name)


def test_abi_version_and_error_plumbing():
    lib = _native.lib()
    assert lib.zc_abi_version() == _native.ABI_VERSION
    assert isinstance(_native.last_error(), str)
    # null handle is rejected without touching a device
    rc = lib.zc_run_log(None, None, None, 0)
    assert rc == _native.ZC_ESTATE
    assert "null" in _native.last_error()


def test_struct_layout_matches_header():
    assert ctypes.sizeof(_native.GraphDesc) == 8 * 5 + 4 * 8
    assert ctypes.sizeof(_native.Stats) == 8 * 3 + 8 * 3 + 8 * 3 + 8 + 8 * 6


def test_host_side_value_errors_match_reference():
    chain = zc.CsrGraph(3, 2, np.array([0, 1, 2, 2]), np.array([1, 2]))
    with pytest.raises(ValueError, match="out of range"):
        zc.bfs(chain, 3)
    with pytest.raises(ValueError, match="out of range"):
        zc.sssp(chain, -1)
    with pytest.raises(ValueError, match="requires edge weights"):
        zc.sssp(chain, 0)
    neg = zc.CsrGraph(3, 2, chain.offsets, chain.edges, weights=np.array([5, -1]))
    with pytest.raises(ValueError, match="non-negative"):
        zc.sssp(neg, 0)
    with pytest.raises(ValueError, match="directed"):
        zc.cc(chain)
    with pytest.raises(ValueError, match="strategy"):
        zc.bfs(chain, 0, "diagonal")


def test_strategy_ids():
    from paper_2006_06890_b200.access import aligned_start, strategy_id
    assert [strategy_id(s) for s in zc.AccessStrategy] == [0, 1, 2]
    assert strategy_id("merged-aligned") == _native.ZC_MERGED_ALIGNED
    # access.py:34-37 examples (test_access.py:70-91)
    assert aligned_start(33, 4) == 32 and aligned_start(4, 8) == 0 and aligned_start(31, 4) == 0


def test_no_cpu_fallback_without_device():
    """On a box without a GPU the product path fails loudly."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    g = zc.generate_uniform(64, 1, 3, seed=1)
    with pytest.raises(RuntimeError):
        zc.bfs(g, 0)


def test_open_emgi_header_errors_match_reference(tmp_path):
    """zc_graph_open_emgi rejects bad files before touching a device, with the
    reference load_csr_binary's ValueErrors (csr.py:204-245)."""
    bad = tmp_path / "bad.emgi"
    bad.write_bytes(b"XXXX" + bytes(40))
    with pytest.raises(ValueError, match="magic"):
        zc.open_emgi(str(bad))
    bad.write_bytes(b"EMGI")
    with pytest.raises(ValueError, match="truncated"):
        zc.open_emgi(str(bad))
    g = zc.with_uniform_weights(zc.generate_uniform(100, 1, 3, seed=1))
    p = tmp_path / "g.emgi"
    zc.store_csr_binary(g, str(p))
    raw = p.read_bytes()
    p.write_bytes(raw[:-5])
    with pytest.raises(ValueError, match="weight array incomplete"):
        zc.open_emgi(str(p))
    p.write_bytes(raw[:4] + (2).to_bytes(4, "little") + raw[8:])
    with pytest.raises(ValueError, match="version"):
        zc.open_emgi(str(p))


def test_open_emgi_rejects_wrapping_header_counts(tmp_path):
    """Untrusted header counts are bounded by the file size before any
    multiplication (a wrapped ne * 4 must not pass the truncation check)."""
    import struct
    for nv, ne in ((4, (1 << 62) + 1), (4, (1 << 64) - 1), ((1 << 61), 2), ((1 << 64) - 1, 0)):
        path = tmp_path / f"bad_{nv}_{ne}.emgi"
        body = struct.pack("<4sIIQQ", b"EMGI", 1, 0, nv, ne) + bytes(8 * 5 + 128)
        path.write_bytes(body)
        with pytest.raises(ValueError, match="truncated"):
            zc.open_emgi(str(path))
