import sys, numpy as np
sys.path.insert(0, "tests"); sys.path.insert(0, ".")
from oracle import oracle
from paper_2107_07866_b200.potential import write_baseline_table
import test_slab as T
from helpers import structure
p = write_baseline_table("/tmp/b.eam")
ref = oracle.Sim(p, box=(8, 7, 10), temperature=600.0, seed=77)
print("box", ref.box)
dom = T.slab_domain(ref, p, 2)
for r in dom.ranks: print("info", r.info, r.n_slots)
dom.prime()
a = structure(T._interior(ref.store()))[0]; b = structure(T.gather(dom, ref))[0]
print(len(a), len(b))
ka, kb = set(a), set(b)
print("only ref", sorted(ka - kb)[:10], len(ka - kb))
print("only dev", sorted(kb - ka)[:10], len(kb - ka))
diff = [k for k in ka & kb if a[k] != b[k]]
print("tag diff", diff[:10], len(diff))
