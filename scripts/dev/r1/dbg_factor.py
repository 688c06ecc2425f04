import sys, faulthandler; faulthandler.enable()
sys.path.insert(0, ".")
import numpy as np, kepgen, oracle
from paper_1710_05134_b200 import Kep
p = kepgen.config(1)
k = Kep.from_pencil(p); k.set_values(p.a, p.b)
print("factor", flush=True); f = k.factor(0.1)
print("info", f.info()["nu"], flush=True)
print("solve", flush=True); x = f.solve(np.ones(p.n))
print("export", flush=True); ex = f.export()
print("close", flush=True); f.close()
print("factor2", flush=True); f2 = k.factor(0.2); print("del", flush=True); del f2
print("done", flush=True)
