"""Anchors bench.py's extrapolated CPU-reference model with one COMPLETE
stock reference slice (VERDICT r1 "Make the measurement honest").

Runs on the host it reports (here or the GPU box, via oracle/_ref):
  measured: the reference's own amplitude_batch -> execute_slice
            (proj/src/sampler.cpp:111-120, src/engine.cpp:182-245) over ONE
            whole slice of the config-3 stand-in, 1 BLAS thread, 1 task;
  model:    bench.py's composite for the same slice on 1 thread (timed plan
            prefix + scaled-down heavy GEMM rate).
Writes profiles/ref_anchor.json; bench.py attaches it to every cpu_baseline.

    python scripts/ref_anchor.py [--config 3s]
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))

import bench  # noqa: E402
import reflib  # noqa: E402


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="3s")
    ap.add_argument("--budget-flops", type=float, default=4e11)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ref_anchor.json"))
    args = ap.parse_args()
    cfg = bench.CONFIGS[args.config]
    plan_text = open(os.path.join(ROOT, cfg["plan"])).read()
    plan = json.loads(plan_text)
    text = bench.circuit_text(cfg, reflib.generate_rqc)
    n = int(text.split()[0])
    reflib.lib().ref_set_blas_threads(1)

    # model on one thread (exactly bench.py's composite)
    nsteps = bench.reference_prefix_steps(plan, args.budget_flops)
    secs, fl = bench.cpu_reference_sample(cfg, nsteps, 1, ntasks=1)
    prefix_rate = fl / secs
    heavy_rate, heavy_desc = (bench.cpu_heavy_gemm_rate(plan, 1) if bench.heavy_unmeasured(plan, nsteps) > 0
                              else (prefix_rate, "no heavy steps beyond the prefix"))
    total = plan["per_slice"]["flops"]
    heavy = bench.heavy_unmeasured(plan, nsteps)
    model_s = heavy / heavy_rate + (total - heavy) / prefix_rate

    # one complete stock slice
    x1 = [0] * n
    for q in plan["open_qubits"]:
        x1[q] = -1
    t0 = time.perf_counter()
    reflib.amplitude_batch(text, plan_text, x1, [0])
    measured_s = time.perf_counter() - t0

    nproc, model = bench.host_cpu()
    out = {"config": cfg["workload"], "slice_flops": total, "measured_s": measured_s, "model_s": model_s,
           "measured_over_model": measured_s / model_s,
           "prefix_rate_gflops": prefix_rate / 1e9, "heavy_rate_gflops": heavy_rate / 1e9, "heavy_desc": heavy_desc,
           "host": {"nproc": nproc, "cpu_model": model},
           "note": "one whole slice through the stock amplitude_batch/execute_slice on 1 thread vs bench.py's "
                   "composite model on 1 thread; >1 means the model is optimistic for the reference"}
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
