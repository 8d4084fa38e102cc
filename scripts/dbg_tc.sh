for d in 0 1 2 4 3 6 7; do
  HGA_TC_DBG=$d python - <<'PY'
import os, torch, json
os.environ["HGA_FITNESS_TC"]="all"
from paper_2208_14961_b200 import engine
from paper_2208_14961_b200._lib import lib
st=torch.cuda.current_stream().cuda_stream
for m in (20,48):
    n=250000
    pop=engine.init_population_device(engine.GAConfig(order=m, population=n//4, seed=1))
    out=torch.empty(n,dtype=torch.int64,device="cuda")
    for _ in range(3): lib.hga_fitness_i8(pop.data_ptr(), n, m, 2, None, out.data_ptr(), None, None, None, None, 0, st)
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): lib.hga_fitness_i8(pop.data_ptr(), n, m, 2, None, out.data_ptr(), None, None, None, None, 0, st)
    e1.record(); e1.synchronize()
    t=e0.elapsed_time(e1)/5/1e3
    print(json.dumps({"dbg": int(os.environ["HGA_TC_DBG"]), "m": m, "us": t*1e6, "evals_per_s": n/t}))
PY
done
