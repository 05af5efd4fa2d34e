import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_1905_00444_b200 as Q
text = Q.generate_rqc(4, 4, 16, 0)
pt = open("configs/config1_plan.json").read()
opn = json.loads(pt)["open_qubits"]
closed = [q for q in range(16) if q not in opn]
wide = Q.widen_plan(text, pt, closed)
eng = Q.Engine(text, wide)
x1s = np.asarray([Q.draw_x1(16, opn, 1, t) for t in range(1024)], dtype=np.int32)
for _ in range(5): eng.amplitude_batches(opn, x1s, [0], bitstrings=False)
def timeit(fn, n=50):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    for _ in range(n): fn()
    torch.cuda.synchronize(); return (time.perf_counter() - t0) / n * 1e3
x1w = [-1] * 16
print("api amplitude_batches ms", timeit(lambda: eng.amplitude_batches(opn, x1s, [0], bitstrings=False)))
eng.prepare(x1w)
print("run+sync ms", timeit(lambda: (eng.run([0], reset=True), eng.synchronize())))
print("run+results ms", timeit(lambda: (eng.run([0], reset=True), eng.results())))
print("results only ms", timeit(lambda: eng.results()))
