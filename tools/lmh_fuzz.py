"""LMH on random finite-support programs (tests/fuzz_programs.py discrete_program) against
their exact GPU enumeration: total variation of the return value's distribution per seed."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from fuzz_programs import discrete_program  # noqa: E402

from paper_2010_08454_b200 import Rng, frontend, infer  # noqa: E402


def main(n_seeds=12):
    for seed in range(n_seeds):
        src = discrete_program(seed)
        ex = dict(infer.run_enumeration(frontend.compile_program(src)).support)
        mc = infer.run_lmh(frontend.compile_program(src.replace("enumerate(model, 100000)", "mcmc(model, 10)")),
                           3000, Rng(seed), chains=512, burn_in=300)
        got = dict(mc.support)
        tv = 0.5 * sum(abs(got.get(k, 0.0) - ex.get(k, 0.0)) for k in set(ex) | set(got))
        print(seed, round(tv, 4), round(mc.stats["acceptance"], 3))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 12)
