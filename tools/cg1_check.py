import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2103_17040_b200 import abi, configs
from oracle import port
cfg = configs.CONFIGS['c3'].resized(4, 64)
os.environ['TS_PCG_CG1'] = '1'
g = abi.Context(cfg.ini(), cfg.ext())
o = port.OracleContext(cfg)
out = g.solve(outer_tol=cfg.outer_tol); ref = o.solve(outer_tol=cfg.outer_tol)
rel = lambda a, b: np.linalg.norm(a - b) / np.linalg.norm(b)
print('sweeps', out['sweeps'], ref['sweeps'], 'relV', rel(out['V'], ref['V']), 'relu', rel(out['u'], ref['u']))
u = np.full(g.n_macro, 0.05); w = np.zeros(g.n_macro)
V, it, _ = g.micro_solve(u, w); oV, oit = o.micro_sweep(u, w)
print('iters maxdiff', np.abs(it - oit).max(), 'relV', rel(V, oV))
