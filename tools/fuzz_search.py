"""Wider differential search than tests/test_frontend_fuzz.py: seeds [a, b) of the random
program generator, GPU log-weights vs the fp64 interpreter; prints failing seeds."""
import math
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
import numpy as np  # noqa: E402

from fuzz_programs import misc_program, program, vector_program  # noqa: E402
from oracle.dsl_eval import Interpreter  # noqa: E402
from paper_2010_08454_b200 import Rng, frontend, infer  # noqa: E402


GEN = {"scalar": program, "vector": vector_program, "misc": misc_program}


def check(seed, gen="scalar"):
    src = GEN[gen](seed)
    m = frontend.compile_program(src)
    post = infer.run_importance(m, 1024, Rng(seed), return_traces=True)
    lw = post.traces["log_weight"].cpu().numpy().astype(float)
    draws = post.traces["draws"].cpu().numpy().astype(float)
    it = Interpreter(src)
    worst = 0.0
    for i in range(0, 1024, 37):
        ref, _ = it.run(draws[i])
        if not math.isfinite(ref):
            if np.isfinite(lw[i]):
                return f"non-finite mismatch at {i}: {lw[i]} vs {ref}"
            continue
        err = abs(lw[i] - ref) / (abs(ref) + 1.0)
        worst = max(worst, err)
        if abs(lw[i] - ref) > 1e-4 * abs(ref) + 1e-4:
            return f"particle {i}: {lw[i]} vs {ref} (draws {draws[i]})"
    return None


def main(a, b, gen="scalar"):
    fails = 0
    for seed in range(a, b):
        try:
            msg = check(seed, gen)
        except Exception as e:  # noqa: BLE001
            msg = f"{type(e).__name__}: {str(e)[:300]}"
        if msg:
            fails += 1
            print(f"seed {seed}: {msg}")
    print(f"seeds {a}..{b}: {fails} failing")


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), sys.argv[3] if len(sys.argv) > 3 else "scalar")
