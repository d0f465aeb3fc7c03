"""Run the importance-sampling kernel a few times (profiling target for ncu)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2010_08454_b200 import Rng, infer, models  # noqa: E402


def main(kind="poly", n=2_000_000_000, reps=3):
    n, reps = int(n), int(reps)
    m = models.PolyRegression.synthetic() if kind == "poly" else models.LinearRegression.synthetic(n_points=1000)
    L = infer.IsLauncher(m, torch.device("cuda", 0))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k in range(reps):
        if k == reps - 1:
            e0.record()
        L.launch(0, n, Rng(1).split(k).key)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{kind}: n={n} {ms:.3f} ms  {n / ms * 1e3:.4g} particles/s")


if __name__ == "__main__":
    main(*sys.argv[1:])
