# Which Bristlecone-70 slices contribute (for the fixture bitstring)?  Then
# the accuracy knobs on config 2 and the config-4 knob sweep.
mkdir -p gpurun_out
python - <<'PY'
import json, numpy as np, sys
sys.path.insert(0, ".")
import paper_1905_00444_b200 as Q
text = open("tests/golden/bristlecone70_circuit.txt").read()
plan = open("configs/config4_bristlecone70_plan.json").read()
x1 = json.load(open("tests/golden/large_bc70.json"))["x1"][0]
with Q.Engine(text, plan) as e:
    e.prepare(x1)
    ids = list(range(256))
    e.run(ids, reset=True, per_slice=True)
    amps, per = e.results(per_slice=True)
nzs = [i for i in ids if abs(per[i][0]) > 0]
print("bc70 nonzero slices among 0..255:", len(nzs), nzs[:16], "amp", amps[0])
json.dump({"nonzero": nzs}, open("gpurun_out/bc70_nonzero.json", "w"))
PY
bash scripts/gpu_r2_acc.sh
bash scripts/gpu_r2_sweep_c4.sh
