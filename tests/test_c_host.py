"""The C ABI drives the generation loop from plain C (examples/qeqea_host.c):
same records and best circuit as the Python facade."""
import shutil
import subprocess

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_c_host_matches_python_engine(tmp_path):
    gcc = shutil.which("gcc") or shutil.which("cc")
    if gcc is None:
        pytest.skip("no C compiler")
    exe = tmp_path / "qeqea_host"
    lib = ROOT / "paper_1809_11134_b200"
    subprocess.run([gcc, "-O2", "-I", str(ROOT / "include"), str(ROOT / "examples" / "qeqea_host.c"),
                    "-L", str(lib), "-lisq", f"-Wl,-rpath,{lib}", "-o", str(exe)], check=True)
    out = subprocess.run([str(exe), "120"], check=True, capture_output=True, text=True).stdout.split("\n")
    rows = [list(map(float, ln.split()[1:])) for ln in out if ln and ln[0].isdigit()]
    tail = [ln for ln in out if ln.startswith("stop")][0].split()

    from paper_1809_11134_b200 import PopulationConfig, QeqeaEngine, target_matrix
    from paper_1809_11134_b200.gates import encode_gates

    eng = QeqeaEngine(PopulationConfig(3, 16, 5, max_generations=120), target_matrix("Toffoli"), 1)
    rec = eng.steps(120)
    assert np.array_equal(np.array(rows), np.stack([rec["gen_best"], rec["gen_mean"], rec["best_fitness"]], 1))
    codes, _ = encode_gates(eng.best_gates, 3)
    assert [int(x) for x in tail[5:]] == list(codes)
    assert float(tail[3]) == eng.best_fitness
