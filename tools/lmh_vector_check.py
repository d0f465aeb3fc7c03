"""LMH vs importance sampling on random programs over drawn vectors with a scalar return
(tests/fuzz_programs.py vector_program): posterior means of the returned value."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from fuzz_programs import vector_program  # noqa: E402

from paper_2010_08454_b200 import Rng, frontend, infer  # noqa: E402


def main(n=16):
    for seed in range(n):
        src = vector_program(seed)
        if not src.rstrip().endswith("importance(model, 1000)") or "  c\n};" in src:
            continue  # scalar returns only
        isd = infer.run_importance(frontend.compile_program(src), 4_000_000, Rng(seed))
        mc = infer.run_lmh(frontend.compile_program(src.replace("importance(model, 1000)", "mcmc(model, 10)")),
                           4000, Rng(seed), chains=1024, burn_in=1000)
        sd = max(isd.stats["var_value"], 1e-12) ** 0.5
        print(seed, "IS", round(isd.mean["value"], 4), "LMH", round(mc.mean["value"], 4), "post sd", round(sd, 4),
              "ess", int(isd.ess), "acc", round(mc.stats["acceptance"], 3))


if __name__ == "__main__":
    main(int(sys.argv[1]) if len(sys.argv) > 1 else 16)
