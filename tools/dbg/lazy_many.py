import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from abft_inputs import make_problem, Fault
from tests.parity_util import gpu_run, oracle_run, key
p = make_problem("cfg3", nx=96, ny=64, nz=20, sweeps=6, nfaults=0, checksums=1)
faults = [Fault(3, z, (5 * z) % 64, (11 * z) % 96, 29) for z in range(20)]
faults += [Fault(5, z, 0, 95, 30) for z in range(0, 20, 3)]
for ns in (3, 4, 5, 6):
    o = oracle_run(p, nsweeps=ns, faults=faults)
    g = gpu_run(p, nsweeps=ns, faults=faults)
    bad = np.flatnonzero(g["u"].view(np.uint32) != o["u"].view(np.uint32))
    print("nsweeps", ns, "bad", bad.size, [np.unravel_index(b, g["u"].shape) for b in bad[:6]])
    gr = sorted(g["records"], key=key); orr = sorted(o["records"], key=key)
    for a, b in zip(gr, orr):
        if a != b:
            print(" G", a); print(" O", b)
    if len(gr) != len(orr): print("len", len(gr), len(orr))
