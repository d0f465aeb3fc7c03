import sys
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
from fuzz_programs import discrete_program
from paper_2010_08454_b200 import Rng, frontend, infer
for seed in range(12):
    src = discrete_program(seed)
    ex = dict(infer.run_enumeration(frontend.compile_program(src)).support)
    mc = infer.run_lmh(frontend.compile_program(src.replace("enumerate(model, 100000)", "mcmc(model, 10)")),
                       3000, Rng(seed), chains=512, burn_in=300)
    got = dict(mc.support)
    tv = 0.5 * sum(abs(got.get(k, 0.0) - ex.get(k, 0.0)) for k in set(ex) | set(got))
    print(seed, round(tv, 4), round(mc.stats["acceptance"], 3))
