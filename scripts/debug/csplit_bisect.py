"""Config 2 slice 0 with split hand-offs restricted to one producer step, vs none."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.getcwd())
import paper_1905_00444_b200 as Q

text = Q.generate_rqc(7, 7, 32, 0)
plan = open("configs/config2_plan.json").read()
x1 = Q.draw_x1(49, json.loads(plan)["open_qubits"], 0, 0)

def run(only):
    if only is None:
        os.environ["QSG_TC_CSPLIT"] = "0"
        os.environ.pop("QSG_TC_CSPLIT_ONLY", None)
    else:
        os.environ["QSG_TC_CSPLIT"] = "1"
        os.environ["QSG_TC_CSPLIT_ONLY"] = str(only)
    with Q.Engine(text, plan, tensor_cores=True) as e:
        e.prepare(x1)
        e.run([0], reset=True, per_slice=True)
        a, _ = e.results()
        lst = [l for l in e.describe().splitlines() if "split" in l]
    return np.asarray(a), lst

ref, _ = run(None)
for st in sys.argv[1:]:
    a, lst = run(st)
    err = np.linalg.norm(a - ref) / np.linalg.norm(ref)
    print(st, f"{err:.3e}", lst, flush=True)
