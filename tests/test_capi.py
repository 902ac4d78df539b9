"""CPU: the C-ABI library builds, loads and exports exactly what
include/hg_b200.h declares; host-side semantics (config defaults, V
derivation, errors) follow the reference. No compute calls without a GPU."""
import ctypes as C
import subprocess

import numpy as np
import pytest

from paper_1907_02900_b200 import _lib


def test_library_loads_and_exports_header_symbols():
    L = _lib.lib()
    declared = _lib.header_functions()
    assert len(declared) >= 15
    for name in declared:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared) <= exported
    assert set(_lib.SIGNATURES) == set(declared)
    assert L.hg_abi_version() == 1


def test_sm100a_only_cubin():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_build_config_defaults_match_reference():
    # core.hpp:30-35 BuildConfig{} and join.hpp:25-28 ProbeOptions{}
    c = _lib.hg_build_config()
    _lib.lib().hg_build_config_init(C.byref(c))
    assert c.load_factor == 1.0 and c.bin_count == 1 << 15 and c.hash_seed == 0
    assert c.variant == 1 and c.stable == 0 and c.vertex_count == 0
    o = _lib.hg_probe_options()
    _lib.lib().hg_probe_options_init(C.byref(o))
    assert o.materialize == 0 and o.pair_cap == 1 << 24 and o.pair_width == 8


def test_derived_vertex_count_and_errors():
    import paper_1907_02900_b200 as hg
    assert [hg.derived_vertex_count(10, l) for l in (1.0, 2.0, 0.5, 4.0)] == [10, 5, 20, 2]
    assert hg.derived_vertex_count(3, 10.0) == 1 and hg.derived_vertex_count(0, 1.0) == 1
    for bad in (0.0, -1.0):
        with pytest.raises(ValueError):
            hg.derived_vertex_count(10, bad)


def test_host_hash_matches_golden(oracle):
    import json, os
    import paper_1907_02900_b200 as hg
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
    for k, s, v, out in g["hash_to_vertex"]:
        assert hg.hash_to_vertex(int(k, 16), int(s, 16), int(v, 16)) == int(out, 16)


def test_invalid_config_rejected_before_device():
    import paper_1907_02900_b200 as hg
    with pytest.raises(ValueError):
        hg.build_v1([1, 2, 3], hg.BuildConfig(load_factor=0.0))
    with pytest.raises(ValueError):
        hg.build_v2([1, 2, 3], hg.BuildConfig(bin_count=0))


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1907_02900_b200 as hg
    with pytest.raises(_lib.HashGraphError) as ei:
        hg.build_v1([1, 2, 3])
    assert ei.value.status == _lib.HG_ECUDA


def test_key_files_match_the_reference(tmp_path, reference):
    """HGKEYS01 (keygen.hpp:97-132): files written by the engine are read by the
    reference and vice versa; format errors raise KeyFileError (host paths only,
    no GPU needed)."""
    import paper_1907_02900_b200 as hg
    rng = np.random.default_rng(5)
    keys = rng.integers(0, 1 << 63, size=100003, dtype=np.uint64)
    keys[:3] = [0, 0xFFFFFFFFFFFFFFFF, 7]
    a = str(tmp_path / "a.keys")
    hg.write_keys(a, keys)
    assert (reference.read_keys(a) == keys).all()
    b = str(tmp_path / "b.keys")
    reference.write_keys(b, keys[:777])
    assert open(a, "rb").read()[:8] == b"HGKEYS01"
    assert (hg.read_keys(b) == keys[:777]).all()
    # u32 in and out (zero-extended on write, range-checked on read)
    small = keys[:50] & np.uint64(0xFFFFFFFF)
    hg.write_keys(b, small.astype(np.uint32))
    assert (reference.read_keys(b) == small).all()
    assert (hg.read_keys(b, key_width=4) == small.astype(np.uint32)).all()
    with pytest.raises(hg.OutOfRange):
        hg.read_keys(a, key_width=4)
    # empty file round trip
    hg.write_keys(b, np.zeros(0, np.uint64))
    assert len(hg.read_keys(b)) == 0 and len(reference.read_keys(b)) == 0
    # format errors (keygen.hpp:117-126)
    bad = tmp_path / "bad.keys"
    for blob in (b"HGKEYS0", b"XXKEYS01" + bytes(8), b"HGKEYS01" + (2).to_bytes(8, "little") + bytes(8),
                 b"HGKEYS01" + (1).to_bytes(8, "little") + bytes(9)):
        bad.write_bytes(blob)
        with pytest.raises(hg.KeyFileError):
            hg.read_keys(str(bad))
    with pytest.raises(hg.KeyFileError):
        hg.read_keys(str(tmp_path / "missing.keys"))
