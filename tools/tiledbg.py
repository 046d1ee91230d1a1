import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2009_13916_b200 import configs
from paper_2009_13916_b200.device import DeviceSystem
from paper_2009_13916_b200.precond import BlockLDUPreconditioner, patterns_for
case = configs.config2(n=64)
s = case.system
ds = DeviceSystem.from_host(s)
pre = BlockLDUPreconditioner.build(ds, patterns=patterns_for(s, "static", "A"), no_fill=True)
r = torch.randn(s.n_unknowns, dtype=torch.float64, device="cuda")
for _ in range(3): y = pre.apply(r)
torch.cuda.synchronize()
