"""Final-build re-run of the 50x50 coarse-key search (2^49 strategies, 2^36 units, dynamic chunks):
value and argmax must equal round 1's byte and 16-bit results (profiles/r01/validate_50x50.json),
and the argmax must attain the value (oracle, from scratch)."""
import json, os, sys, time
sys.path.insert(0, os.getcwd())
import oracle
import paper_2503_21596_b200 as L
from paper_2503_21596_b200 import synth
ref = json.load(open("profiles/r01/validate_50x50.json"))
M = synth.random_matrix(50, 50, 150)
t = time.time()
v, arg = L.compute(M)
dt = time.time() - t
st = L.last_stats()
out = {"value": int(v), "seconds": dt, "walk_ms": st["walk_ms"], "units": st["units"],
       "same_as_r01_byte": int(v) == ref["auto"]["value"] and list(map(int, arg)) == ref["auto"]["argmax"],
       "same_as_r01_pair16": int(v) == ref["pair16"]["value"] and list(map(int, arg)) == ref["pair16"]["argmax"],
       "oracle_value_of_argmax": int(oracle.value(M, arg))}
print(json.dumps(out))
