"""A/B of the SMC run launched eagerly vs as one captured CUDA graph (same process, same runner
sizes, no timing events): per-run device time by CUDA events around whole runs."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2010_08454_b200 import Rng, models, smc  # noqa: E402


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
    T = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
    reps = 4
    m = models.HiddenMarkovModel.synthetic(S=50, T=T, seed=0)
    for graph in (False, True, False, True):
        r = smc.SmcRunner(m, n, Rng(1), steps=T, graph=graph)
        r.launch()  # warm-up (and capture)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k in range(reps):
            r.reseed(Rng(1).split(k))
            r.launch()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        print(f"n={n} T={T} graph={graph}: {ms:.2f} ms per run, {T / ms * 1e3:.1f} steps/s")
        del r


if __name__ == "__main__":
    main()
