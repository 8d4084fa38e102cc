"""All-variant fitness (F1 + F2 + ORTH + SQ, engine.penalties) at orders 36 / 40:
default routing (tensor-core kernel for several variants) vs XOR+POPC
(HGA_FITNESS_TC=0 in a subprocess), 10^6 matrices, and results identical."""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CODE = r"""
import sys, json, torch, numpy as np
sys.path.insert(0, %r)
from paper_2208_14961_b200 import engine
from paper_2208_14961_b200._lib import lib
out = []
for m in (36, 40):
    n = 1_000_000
    pop = engine.init_population_device(engine.GAConfig(order=m, population=n // 4, seed=7))
    r = [torch.empty(n, dtype=torch.int64, device="cuda") for _ in range(4)]
    sp = torch.cuda.current_stream().cuda_stream
    fn = lambda: lib.hga_fitness_i8(pop.data_ptr(), n, m, 15, r[0].data_ptr(), r[1].data_ptr(), r[2].data_ptr(),
                                    r[3].data_ptr(), None, None, 0, sp)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); fn(); fn(); fn(); e.record(); e.synchronize()
    t = s.elapsed_time(e) / 3 / 1e3
    h = int(sum(int(x.sum().item()) * (i + 1) for i, x in enumerate(r)))
    out.append({"m": m, "evals_per_s": n / t, "checksum": h})
print(json.dumps(out))
""" % str(ROOT)
res = {}
for name, env in (("default", {}), ("xor_popc", {"HGA_FITNESS_TC": "0"})):
    p = subprocess.run([sys.executable, "-c", CODE], env={**os.environ, **env}, capture_output=True, text=True)
    res[name] = json.loads(p.stdout.strip().splitlines()[-1])
for a, b in zip(res["default"], res["xor_popc"]):
    print(json.dumps({"m": a["m"], "all_variants_evals_per_s_default": a["evals_per_s"],
                      "all_variants_evals_per_s_xor_popc": b["evals_per_s"], "identical": a["checksum"] == b["checksum"]}))
