"""The C-ABI library loads on a CPU-only host, exports every entry point the public
header declares, and fails loudly (TS_ERR_CUDA) instead of falling back to the CPU.
The INI/expression front-end (host C++) reports configuration errors with the
reference's messages before any device work."""
import os
import re

import pytest

from paper_2103_17040_b200 import abi, configs

HEADER = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include", "twoscale_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[\w\s\*]+?\b(ts_\w+)\s*\(", text, flags=re.M)))


def test_header_symbols_exported():
    lib = abi.lib()
    names = declared_symbols()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    assert sorted(abi.EXPORTS) == names
    assert lib.ts_abi_version() == 3


@pytest.mark.skipif(abi.lib().ts_device_ok() == 1, reason="GPU present")
def test_no_cpu_fallback_without_device():
    cfg = configs.CONFIGS["c1"].resized(2, 2)
    with pytest.raises(abi.TwoScaleError) as e:
        abi.Context(cfg.ini(), cfg.ext())
    assert e.value.status == abi.TS_ERR_CUDA
    assert "no CUDA device" in str(e.value)
    with pytest.raises(abi.TwoScaleError):
        abi.cg_solve([0, 1], [0], [1.0], [1.0], [0.0], 1e-10, 10)


@pytest.mark.parametrize("ini, msg", [
    ("[macro]\nn0 = 2\n", "missing required keys: macro.n1 micro.n0 micro.n1 micro.zeta0 micro.zeta1"),
    (configs.CONFIGS["c1"].ini().replace("[solver]", "[solver]\nbogus = 1"), "[solver] unknown key 'bogus'"),
    (configs.CONFIGS["c1"].ini().replace("gamma_o =", "gamma_o = left"), "[micro] side 'left' must be assigned"),
    (configs.CONFIGS["c1"].ini().replace("zeta0 = y0", "zeta0 = foo + y0"), "[micro] zeta0: unknown identifier 'foo'"),
    (configs.CONFIGS["c1"].ini().replace("fu = 1", "fu = y0"), "[parameters] fu: expression must not depend on y0/y1"),
    (configs.CONFIGS["c1"].ini() + "[weird]\n", "unknown section [weird]"),
    (configs.CONFIGS["c1"].ini().replace("n0 = 16", "n0 = 1.5", 1), "[macro] n0: expected an integer"),
])
def test_config_errors_match_reference(ini, msg, ref_mod):
    with pytest.raises(abi.ConfigError) as e:
        abi.Context(ini)
    assert msg in str(e.value)
    with pytest.raises(ref_mod.RefError) as r:
        ref_mod.RefContext(ini, 1)
    assert msg in str(r.value)


def test_reference_api_caller_links_against_the_library():
    """oracle/ref_harness.cpp (reference public API only) compiled unchanged against
    include/twoscale and linked to libtwoscale_b200.so (oracle/_mirror) resolves every symbol;
    no GPU call is made here."""
    import ctypes
    from oracle import ref
    path = ref.mirror().LIB_PATH
    assert os.path.exists(path), "make -C oracle mirror"
    L = ctypes.CDLL(path)
    for name in ("ref_create", "ref_solve", "ref_cg_solve", "ref_build_cache", "ref_validate_diffeo",
                 "ref_check_assumption6", "ref_micro_sweep", "ref_write_vtk", "ref_hardware_threads"):
        assert hasattr(L, name), name
    assert L.ref_hardware_threads() >= 1  # resolve_worker_count(0): host-only, no device needed


def test_array_arguments_are_validated():
    """Caller-supplied arrays cross the C ABI as raw pointers: wrong dtype, shape or
    contiguity must raise before any pointer is formed (advisor round 1)."""
    import numpy as np
    ok = np.zeros((3, 4))
    assert abi._out(ok, (3, 4), "V") is ok
    for bad in (np.zeros((3, 4), np.float32), np.zeros((4, 3)), np.zeros((3, 8))[:, ::2], np.zeros(12)):
        with pytest.raises(ValueError):
            abi._out(bad, (3, 4), "V")
    ro = np.zeros((3, 4))
    ro.flags.writeable = False
    with pytest.raises(ValueError):
        abi._out(ro, (3, 4), "V")
    assert abi._in([1, 2, 3], 3, "u").dtype == np.float64
    with pytest.raises(ValueError):
        abi._in(np.zeros(4), 3, "u")
    with pytest.raises(ValueError):
        abi.cg_solve(np.array([0, 1, 2]), np.array([0]), np.array([1.0]), np.ones(2), np.zeros(2), 1e-10, 10)
