"""The C-ABI library loads and exports every symbol include/qsg.h declares;
compute entry points fail loudly (no CPU fallback) without a GPU."""
import ctypes
import subprocess

import pytest

import paper_1905_00444_b200 as Q
from conftest import has_gpu


def test_library_exports_every_header_symbol():
    L = Q.lib()
    names = Q.exported_symbols()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing


def test_library_targets_sm100a_only():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", Q.LIB_PATH], capture_output=True, text=True)
    assert out.returncode == 0
    assert "sm_100a" in out.stdout


@pytest.mark.skipif(has_gpu(), reason="checks the no-GPU failure path")
def test_compute_without_gpu_fails_loudly():
    import numpy as np
    with pytest.raises(Q.QsgError) as e:
        Q.transpose(np.zeros((2, 2), np.complex64), [1, 0])
    assert e.value.kind == "cuda"
    with pytest.raises(Q.QsgError):
        Q.Engine(Q.generate_rqc(2, 2, 2, 0), kind=Q.PLAN_GREEDY, open_qubits=[3])
