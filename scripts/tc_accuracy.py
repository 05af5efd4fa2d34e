"""Accuracy study of the K2 kernels (run on a GPU box):
  * tcgen05 3xTF32 vs FP32 SIMT vs fp64 across reduction lengths k;
  * config 2 (7x7, 1+32+1, 1024-amp batch) amplitudes, tensor-core engine vs
    SIMT engine (two independent GEMM implementations at full size).
Writes a JSON summary to gpurun_out/tc_accuracy.json."""
import json
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1905_00444_b200 as Q  # noqa: E402


def gemm_err(m, n, k, seed=0, scale_spread=False):
    g = torch.Generator().manual_seed(seed)
    A = torch.complex(torch.rand(m, k, generator=g) - 0.5, torch.rand(m, k, generator=g) - 0.5)
    B = torch.complex(torch.rand(k, n, generator=g) - 0.5, torch.rand(k, n, generator=g) - 0.5)
    if scale_spread:
        A = A * torch.exp2(torch.randint(-8, 8, (m, k), generator=g).float())
    want = A.to(torch.complex128) @ B.to(torch.complex128)
    dA, dB = A.cuda(), B.cuda()
    out = {}
    wsb = int(Q.lib().qsg_cgemm_tc_workspace_bytes(m, n, k, 0))
    ws = torch.empty(max(wsb, 16), dtype=torch.uint8, device="cuda")
    for name, fn in (("tc", lambda c: Q.lib().qsg_cgemm_tc_dev(dA.data_ptr(), dB.data_ptr(), c.data_ptr(), m, n, k, 0,
                                                               ws.data_ptr(), wsb, None)),
                     ("simt", lambda c: Q.lib().qsg_cgemm_dev(dA.data_ptr(), dB.data_ptr(), c.data_ptr(), m, n, k, 0, 0, None))):
        c = torch.zeros(m, n, dtype=torch.complex64, device="cuda")
        Q._check(fn(c))
        torch.cuda.synchronize()
        got = c.cpu().to(torch.complex128)
        out[name] = float((got - want).abs().norm() / want.abs().norm())
    # plain complex64 torch (cuBLAS) as a yardstick
    c = (dA @ dB).cpu().to(torch.complex128)
    out["cublas_c64"] = float((c - want).abs().norm() / want.abs().norm())
    return out


def main():
    res = {"gemm": []}
    for k in (16, 64, 256, 1024, 4096, 16384, 65536):
        for spread in (False, True):
            e = gemm_err(128, 128, k, seed=k, scale_spread=spread)
            e.update({"m": 128, "n": 128, "k": k, "spread": spread})
            res["gemm"].append(e)
            print(e, flush=True)
    # full-size: config 2, TC engine vs SIMT engine, same x1
    text = Q.generate_rqc(7, 7, 32, 0)
    plan = open(os.path.join(ROOT, "configs", "config2_plan.json")).read()
    opn = json.loads(plan)["open_qubits"]
    x1 = Q.draw_x1(49, opn, 0, 0)
    amps = {}
    for tc in (True, False):
        t0 = time.time()
        with Q.Engine(text, plan, tensor_cores=tc) as e:
            _, a = e.amplitude_batch(x1, [0, 1])
        amps[tc] = a
        print("engine tc=%s %.2fs" % (tc, time.time() - t0), flush=True)
    a, b = amps[True], amps[False]
    res["config2_tc_vs_simt"] = {
        "rel_l2": float(np.linalg.norm(a - b) / np.linalg.norm(b)),
        "max_rel_abs": float(np.max(np.abs(np.abs(a) - np.abs(b)) / np.abs(b))),
        "fidelity": float(abs(np.vdot(a, b)) ** 2 / (np.vdot(a, a).real * np.vdot(b, b).real)),
        "norm_sq_times_2n": float(np.vdot(b, b).real * 2 ** 49 / 1024),
    }
    print(res["config2_tc_vs_simt"], flush=True)
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    with open(os.path.join(ROOT, "gpurun_out", "tc_accuracy.json"), "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
