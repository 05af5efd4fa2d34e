"""The C-ABI library loads and exports every symbol include/qsg.h declares;
compute entry points fail loudly (no CPU fallback) without a GPU."""
import ctypes
import os
import subprocess

import pytest

import paper_1905_00444_b200 as Q
from conftest import ROOT, has_gpu


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


REF_INCLUDE = "/root/reference/proj/include"


@pytest.mark.skipif(not os.path.isdir(REF_INCLUDE), reason="reference tree not present (GPU box)")
def test_integration_shim_builds_against_reference_headers(tmp_path):
    """the C++ shim a reference maintainer adds
    (integration/qsg_backend.hpp) compiles against the reference's own qsim
    headers, links against libqsg.so, and -- without a GPU -- fails loudly
    through the reference's exception types (no CPU fallback)."""
    import shutil
    import subprocess
    gxx = shutil.which("g++", path="/usr/bin") or "g++"
    src = tmp_path / "shim_main.cpp"
    src.write_text(
        '#include "qsg_backend.hpp"\n'
        "#include <cstdio>\n"
        "int main() {\n"
        '  qsim::Tensorf a({"i", "k"}, {2, 2}), b({"k", "j"}, {2, 2});\n'
        "  try {\n"
        '    auto c = qsim::qsg_backend::contract_normalized(a, b, {"i", "j"}, nullptr);\n'
        '    std::printf("ran %lld\\n", (long long)c.volume());\n'
        "    return 0;\n"
        "  } catch (const std::runtime_error& e) {\n"
        '    std::printf("error: %s\\n", e.what());\n'
        "    return 3;\n"
        "  }\n"
        "}\n")
    exe = tmp_path / "shim_main"
    lib_dir = os.path.join(ROOT, "paper_1905_00444_b200")
    jsoninc = "/opt/prime-rl/.venv/lib/python3.12/site-packages/include/cudnn_frontend/thirdparty"
    cmd = [gxx, "-std=c++20", "-O1", "-I", os.path.join(ROOT, "integration"), "-I", os.path.join(ROOT, "include"),
           "-I", REF_INCLUDE, "-I", os.path.join(ROOT, "oracle", "shim"), "-I", jsoninc, str(src), "-o", str(exe),
           "-L", lib_dir, "-lqsg", f"-Wl,-rpath,{lib_dir}"]
    subprocess.run(cmd, check=True, capture_output=True)
    res = subprocess.run([str(exe)], capture_output=True, text=True, timeout=120)
    if has_gpu():
        assert res.returncode == 0, res.stdout + res.stderr
    else:
        assert res.returncode == 3 and "CUDA" in res.stdout, res.stdout + res.stderr
