"""Find where a device LGA run first departs from the oracle (s2, fp64fast)."""
import json, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle
from paper_2410_10447_b200 import BASELINE, SINGLE, Device, LgaSettings
from paper_2410_10447_b200._abi import Instance

raw = json.load(open("tests/golden/instances.json"))["s2"]
inst = Instance(np.array(raw["atoms"]), np.array(raw["torsion"]), np.array(raw["sites"]), raw["n_rot"])
port = Oracle("port")
dev = Device(0)
s = LgaSettings()
seeds = np.arange(40, dtype=np.uint64) + np.uint64(4242)
g1 = dev.lga_run_batch(inst, BASELINE, SINGLE, s, seeds)
g2 = dev.lga_run_batch(inst, BASELINE, SINGLE, s, seeds)
print("deterministic:", all(a.best_energy == b.best_energy and a.evaluations == b.evaluations for a, b in zip(g1, g2)))
for sd, g in zip(seeds, g1):
    c = port.lga_run(inst, BASELINE, SINGLE, s, int(sd))
    if g.best_energy == c["best_energy"] and g.evaluations == c["evaluations"]:
        continue
    print("seed", int(sd), "gpu", g.best_energy, g.evaluations, "cpu", c["best_energy"], c["evaluations"])
    for k, (a, b) in enumerate(zip(g.runs, c["runs"])):
        if a != tuple(b):
            print(" first differing LS record", k, "gpu", a, "cpu", b)
            break
