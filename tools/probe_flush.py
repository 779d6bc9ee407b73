import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, ".")
import torch
from paper_2201_03611_b200 import emit_cuda, programs
from paper_2201_03611_b200.run import Executable
sys.path.insert(0, "tools")
from probe_bw import timeit
c = programs.compile_config("dot")
code = emit_cuda(c.unit)
fl = torch.empty(64 << 20, device="cuda"); sw = torch.ones(64 << 20, device="cuda"); sink = torch.empty((), device="cuda")
big = torch.empty(128 << 20, device="cuda")
flushes = {
  "zero+sum": lambda: (fl.zero_(), torch.sum(sw, dim=0, out=sink)),
  "zero only": lambda: fl.zero_(),
  "sum only": lambda: torch.sum(sw, dim=0, out=sink),
  "none": lambda: None,
  "sleep": lambda: torch.cuda._sleep(200000),
}
for lg in (23, 24, 25):
    n = 1 << lg
    exe = Executable(code, {"n": n})
    a = torch.rand(n, device="cuda"); b = torch.rand(n, device="cuda"); out = torch.empty(1, device="cuda")
    bound = exe.bind({"a": a, "b": b, "output": out})
    def two():
        bound(); bound()
    for k, f in flushes.items():
        m1 = timeit(bound, f)[0]; m2 = timeit(two, f)[0]
        print(f"2^{lg} flush={k:10s}: one {m1*1e3:6.1f} us  two {m2*1e3:6.1f} us  second {1e3*(m2-m1):6.1f} us", flush=True)
