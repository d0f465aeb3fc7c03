"""The paper's benchmark table (§5.1) on one B200: each examples/*.cup program compiled
once (NVRTC) and run 10 times at the paper's sizes — 2 million samples for importance sampling,
100 thousand for MCMC (100 chains x 1000 steps), the whole path space for enumeration — wall
clock of the public call (posterior on the host), median of the repeats."""
import json
import statistics
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2010_08454_b200 import Rng, frontend, infer  # noqa: E402

EX = Path(__file__).resolve().parent.parent / "examples"


def run(m, seed):
    if m.engine == "importance":
        return infer.run_importance(m, 2_000_000, Rng(seed)), 2_000_000
    if m.engine == "mcmc":
        return infer.run_lmh(m, 1000, Rng(seed), chains=100), 100_000
    post = infer.run_enumeration(m)
    return post, post.n


def main():
    out = []
    for f in sorted(EX.glob("*.cup")):
        t0 = time.perf_counter()
        m = frontend.compile_program(f.read_text())
        run(m, 0)  # NVRTC build + module load + first launch
        torch.cuda.synchronize()
        t_first = time.perf_counter() - t0
        times = []
        for k in range(10):
            t0 = time.perf_counter()
            _, n = run(m, k + 1)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        med = statistics.median(times)
        rec = {"program": f.stem, "engine": m.engine, "samples": n, "median_s": med,
               "stdev_s": statistics.stdev(times), "samples_per_s": n / med, "first_run_s": t_first}
        out.append(rec)
        print(json.dumps(rec))
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/corpus.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
