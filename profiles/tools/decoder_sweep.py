"""Decoder sweep (C5) on a synthetic instance: K2 random chromosomes, K1 launches timed with events.

    python profiles/tools/decoder_sweep.py J S M [n]

M: one machine count for every stage ("8"), a comma list per stage, or "syn" for the bench's
synthetic convention (M[s] in [2, 8] from Rng(1000 + J*S)).
"""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.environ.get("FFSGA_PKG_ROOT") or ROOT)
import numpy as np
from paper_1903_10722_b200 import capi, generate_instance, estimate_emax, instance_arrays
J, S = int(sys.argv[1]), int(sys.argv[2])
if sys.argv[3] == "syn":
    sys.path.insert(1, ROOT)
    from bench import synthetic_machines
    Ms = synthetic_machines(J, S)
else:
    Ms = [int(x) for x in sys.argv[3].split(",")]
Ms = Ms * S if len(Ms) == 1 else Ms
n = int(sys.argv[4]) if len(sys.argv) > 4 else 1 << 18
d = generate_instance(jobs=J, stages=S, machines=Ms, weight=100.0, seed=7)
ci = capi.Instance.from_data(instance_arrays(d), estimate_emax(d), 0)
b = capi.Batch(ci, n)
b.fill_random(99, 0, n)
for _ in range(2):
    b.evaluate(n)
b.sync()
ms = []
for _ in range(5):
    b.evaluate(n)
    ms.append(b.last_eval_ms())
obj, _ = b.results(n)
print(f"J={J} S={S} M={sys.argv[3]} G={os.environ.get('FFSGA_EVAL_G','auto')} n={n}: {n/np.median(ms)*1e3/1e6:.3f} M evals/s  chk={np.sum(obj):.6e}")
