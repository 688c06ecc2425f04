import sys, os, time
sys.path.insert(0, '.')
os.environ['KEP_DEBUG'] = '1'
import numpy as np, kepgen, oracle
from paper_1710_05134_b200 import Kep
p = kepgen.config(1)
A, B = p.dense('a'), p.dense('b')
w = oracle.eigvals_pencil(A, B)
sig = kepgen.uniform_shifts(w[0], w[-1], 32)
for variant in (0, 1):
    k = Kep.from_pencil(p, pivot_u=0.5, kernel_variant=variant, max_batch=1)
    k.set_values(p.a, p.b)
    for i in range(4):
        t = time.time()
        st, nu, info = k.inertia(sig[i])
        print(variant, i, st, nu, oracle.nu_eig(A, B, sig[i], eigvals=w), info.n_delayed, k.analysis()['delay_slack'], time.time() - t, flush=True)
