"""The reference's own drivers relinked onto the B200 contraction
(VERDICT r1 item 7).

oracle/_ref/libqsim_relink.so is the UNMODIFIED reference library with
src/engine.cpp compiled under integration/qsg_relink.hpp, so the
reference's amplitude_batch -> execute_slice step loop (src/sampler.cpp:
111-120, src/engine.cpp:182-245) runs every contract_ttgt through
qsg_contract (libqsg.so) on the GPU.  Its config-1 batches must equal the
stock reference's (tests/golden/amplitudes.npz, from oracle/_ref/
libqsim_ref.so) within the reference's TTGT tolerance, with bit-identical
bitstrings."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

pytestmark = pytest.mark.gpu

RELINK = os.path.join(ROOT, "oracle", "_ref", "libqsim_relink.so")

_CHILD = r"""
import hashlib, json, os, sys
sys.path.insert(0, os.path.join(sys.argv[1], "oracle"))
import reflib, qsim_oracle as O
text = reflib.generate_rqc(4, 4, 16, 0)
plan = open(os.path.join(sys.argv[1], "configs", "config1_plan.json")).read()
out = []
for i in range(4):
    x1 = O.draw_x1(16, list(range(10, 16)), 0, i)
    bits, amps = reflib.amplitude_batch(text, plan, x1, [0])
    out.append({"sha": hashlib.sha256("".join(bits).encode()).hexdigest(),
                "re": amps.real.tolist(), "im": amps.imag.tolist()})
maps = open("/proc/self/maps").read()
print(json.dumps({"batches": out, "libqsg": "libqsg.so" in maps, "relink": "libqsim_relink.so" in maps}))
"""


@pytest.mark.skipif(not os.path.exists(RELINK), reason="oracle/_ref/libqsim_relink.so not built (make -C oracle)")
def test_relinked_reference_config1_batches(gpu):
    env = dict(os.environ, QSIM_REF_LIB=RELINK)
    res = subprocess.run([sys.executable, "-c", _CHILD, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stderr[-2000:]
    got = json.loads(res.stdout.strip().splitlines()[-1])
    assert got["libqsg"] and got["relink"], "the relinked reference did not load libqsg.so"
    am = np.load(os.path.join(GOLDEN, "amplitudes.npz"))
    meta = json.load(open(os.path.join(GOLDEN, "amplitudes.json")))
    for i, b in enumerate(got["batches"]):
        assert b["sha"] == meta["config1"][i]["bits_sha"]
        amps = np.asarray(b["re"]) + 1j * np.asarray(b["im"])
        ref = am[f"cfg1_amps{i}"]
        assert np.linalg.norm(amps - ref) / np.linalg.norm(ref) < 1e-5, i
