"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/isq.h declares, the ctypes table matches, and the host-side Philox
core equals numpy's Philox."""
import ctypes
import re

import numpy as np
import pytest

from conftest import ROOT

HEADER = ROOT / "include" / "isq.h"


def declared_symbols():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(isq_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    from paper_1809_11134_b200 import _lib

    lib = _lib.load()
    syms = declared_symbols()
    assert len(syms) >= 5
    for s in syms:
        assert hasattr(lib, s), s
    assert set(syms) == set(_lib.SIGNATURES), set(syms) ^ set(_lib.SIGNATURES)
    assert lib.isq_abi_version() == 2


@pytest.mark.parametrize("key", [(0, 1, 0, 0, 0), (7, 3, 12, 999, 0), (2**63 + 5, 8, 2**40, 3, 17)])
def test_host_philox_matches_numpy(key):
    from paper_1809_11134_b200 import _lib

    lib = _lib.load()
    seed, dom, gen, idx, sub = key
    ref = np.random.Philox(key=np.array([seed, dom], dtype=np.uint64),
                           counter=np.array([0, gen, idx, sub], dtype=np.uint64))
    raw = ref.random_raw(12)
    out = np.zeros(4, dtype=np.uint64)
    for b in range(3):
        lib.isq_philox_block(seed, dom, gen, idx, sub, b + 1, out.ctypes.data_as(ctypes.c_void_p))
        assert list(out) == list(raw[4 * b:4 * b + 4])


def test_product_package_does_not_import_oracle():
    pkg = ROOT / "paper_1809_11134_b200"
    for p in pkg.rglob("*.py"):
        assert "oracle" not in re.findall(r"^\s*(?:from|import)\s+(\w+)", p.read_text(), flags=re.M), p


@pytest.mark.parametrize("field,value", [("number_of_wires", 1), ("size_of_individual", 0),
                                         ("probability_of_mutation", 1.5), ("n_meas", 0),
                                         ("world", 9), ("rank", 3), ("precision", 7)])
def test_qeqea_create_validates_before_touching_a_device(field, value):
    """PopulationConfig validation (engine.py:45-63) and the sharding /
    precision checks run in the C ABI before any CUDA call, so they hold on a
    CPU-only host: ISQ_ERR_CONFIG and a message."""
    from paper_1809_11134_b200 import _lib

    lib = _lib.load()
    kw = dict(number_of_wires=3, size_of_individual=8, size_of_population=5, probability_of_mutation=0.3,
              mutation_range=0.78, n_meas=1, rank=0, max_generations=10, target_fitness=0.999, seed=1,
              world=1, precision=0)
    if field == "rank":
        kw["world"] = 2
    kw[field] = value
    conf = _lib.QeqeaConfig(**kw)
    T = np.eye(8, dtype=np.complex128)
    h = ctypes.c_void_p()
    st = lib.isq_qeqea_create(ctypes.byref(conf), T.ctypes.data_as(ctypes.c_void_p), 0, 4, ctypes.byref(h))
    assert st == _lib.ISQ_ERR_CONFIG
    assert h.value is None
    assert lib.isq_last_error()


def test_unsupported_shapes_are_reported_not_computed():
    """n = 14 is a valid reference configuration once its memory_cap_entries
    is raised above the default 2^26 (engine.py:43,60-63); the device build
    stops at the default cap (n = 13): ISQ_ERR_UNSUPPORTED ->
    ConfigurationError, never a CPU fallback."""
    from paper_1809_11134_b200 import _lib
    from paper_1809_11134_b200.errors import ConfigurationError

    lib = _lib.load()
    conf = _lib.QeqeaConfig(number_of_wires=14, size_of_individual=8, size_of_population=5,
                            probability_of_mutation=0.3, mutation_range=0.78, n_meas=1, rank=0,
                            max_generations=10, target_fitness=0.999, seed=1, world=1, precision=0)
    T = np.eye(2, dtype=np.complex128)  # never read: validation fails first
    h = ctypes.c_void_p()
    st = lib.isq_qeqea_create(ctypes.byref(conf), T.ctypes.data_as(ctypes.c_void_p), 0, 4, ctypes.byref(h))
    assert st == _lib.ISQ_ERR_UNSUPPORTED
    with pytest.raises(ConfigurationError):
        _lib.check(st)
    codes, thetas = np.zeros(1, np.uint8), np.zeros(1)
    fit = np.zeros(1)
    st = lib.isq_fitness_batch_ex(14, 1, 1, _lib.ptr(codes), _lib.ptr(thetas), T.ctypes.data_as(ctypes.c_void_p),
                                  _lib.ptr(fit), 0, 0)
    assert st == _lib.ISQ_ERR_UNSUPPORTED


def test_null_handles_are_rejected():
    from paper_1809_11134_b200 import _lib

    lib = _lib.load()
    assert lib.isq_qeqea_begin_batch(None) == _lib.ISQ_ERR_CONFIG
    assert lib.isq_ga_begin_batch(None) == _lib.ISQ_ERR_CONFIG
    assert b"null" in lib.isq_last_error()
    assert lib.isq_qeqea_destroy(None) == _lib.ISQ_OK


def test_c_host_example_compiles_against_the_header(tmp_path):
    """examples/qeqea_host.c builds against include/isq.h + libisq.so with a
    plain C compiler (no CUDA or torch headers in the ABI)."""
    import shutil
    import subprocess

    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        pytest.skip("no C compiler")
    lib = ROOT / "paper_1809_11134_b200"
    subprocess.run([gcc, "-std=c99", "-Wall", "-Werror", "-I", str(ROOT / "include"),
                    str(ROOT / "examples" / "qeqea_host.c"), "-L", str(lib), "-lisq", f"-Wl,-rpath,{lib}",
                    "-o", str(tmp_path / "qeqea_host")], check=True)


def test_encoding_module_mirrors_the_reference_names_without_a_device():
    """encoding.py's public names, constants and argument checks (no device
    call: the Generator refusal and the nMeas check come first)."""
    import math

    import numpy as np

    from paper_1809_11134_b200 import encoding as E
    from paper_1809_11134_b200.errors import ConfigurationError

    for name in ("TWO_PI", "SU3_RANGES", "SU3Params", "read_angle", "mutate_angle", "random_angle", "random_qutrit",
                 "born_probabilities", "measure_qutrit", "estimate_axis", "su3_operator", "mutate_qutrit"):
        assert hasattr(E, name), name
    assert E.TWO_PI == 2.0 * math.pi
    assert np.array_equal(E.SU3_RANGES, np.array([math.pi / 2] * 3 + [2.0 * math.pi] * 5))
    assert E.SU3Params().theta1 == 0.0 and len(E.SU3Params.__dataclass_fields__) == 8
    assert E.read_angle(1.25) == 1.25
    with pytest.raises(TypeError):
        E.mutate_angle(1.0, 0.5, 0.7, np.random.default_rng(1))
    with pytest.raises(TypeError):
        E.mutate_qutrit(np.array([1, 0, 0], dtype=complex), 0.5, np.random.default_rng(1))
    with pytest.raises(ConfigurationError):
        E.estimate_axis(np.array([1, 0, 0], dtype=complex), 0, E.CounterStreams(1))
