import sys; sys.path.insert(0,'/root/repo')
import numpy as np, oracle
import paper_2208_14961_b200 as hga
from paper_2208_14961_b200 import engine
for m, fit, nc, nr in [(12,'f2',2,3),(12,'f2',1,2),(20,'f2',2,3),(28,'f2',2,3),(12,'f2',4,2)]:
    cfg = engine.GAConfig(order=m, population=300, seed=11, fitness=fit, mutation_cols=nc, mutation_row_pairs=nr)
    st = hga.initial_state(cfg)
    for s in range(3):
        before = st.population.copy()
        hga.step(st)
        pop = st.population
        want = oracle.evaluate(pop, fit)
        bad = np.nonzero(st.fitness != want)[0]
        print(m, nc, nr, s, 'mismatch', len(bad), bad[:10], 'N', 300)
