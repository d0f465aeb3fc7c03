"""Run the many-chain MH kernel once (profiling target)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2010_08454_b200 import Rng, infer, models  # noqa: E402


def main(chains=4096, steps=2000, reps=2):
    m = models.GaussianMixture.synthetic(n_points=10_000)
    for k in range(int(reps)):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        r = infer.run_lmh(m, int(steps), Rng(1).split(k), chains=int(chains))
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        print(f"mh: {chains} chains x {steps} steps: {ms:.2f} ms  {int(chains) * int(steps) / ms * 1e3:.4g} chain-steps/s acc={r.acceptance:.3f}")


if __name__ == "__main__":
    main(*sys.argv[1:])
