"""Time the SMC filter on one GPU: per-step device time and effective HBM bandwidth."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2010_08454_b200 import Rng, models, smc  # noqa: E402


def main(n=100_000_000, T=200):
    m = models.HiddenMarkovModel.synthetic(S=50, T=T)
    r = smc.SmcRunner(m, n, Rng(1), steps=T)
    r.init()
    for t in range(5):
        r.step(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for t in range(5, T):
        r.step(t)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / (T - 5)
    res = r.result()
    out = {"n": n, "steps_timed": T - 5, "ms_per_step": ms, "steps_per_s": 1e3 / ms,
           "particle_steps_per_s": n * 1e3 / ms, "alg_GBps_at_14B": 14 * n / (ms / 1e3) / 1e9,
           "log_z": res.log_z, "ess_min": float(res.ess.min())}
    print(json.dumps(out))


if __name__ == "__main__":
    main(*(int(a) for a in sys.argv[1:]))
