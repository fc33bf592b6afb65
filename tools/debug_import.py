import sys, time
t0 = time.time()
def p(m): print(f"{time.time()-t0:7.2f}s {m}", flush=True)
p("start")
import numpy
p("numpy")
import torch
p("torch")
p(f"cuda avail {torch.cuda.is_available()}")
torch.zeros(1, device="cuda")
p("torch cuda init")
sys.path.insert(0, ".")
from paper_2108_08845_b200 import _native as nat
p("import pkg")
L = nat.lib()
p(f"lib loaded v{L.psvd_version()}")
c = nat.context(torch.device("cuda", 0))
p("ctx created")
