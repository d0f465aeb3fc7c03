"""Small runs of the paths smoke() does not cover, for compute-sanitizer: SMC graph replay and
snapshot/restore, compiled categorical / enumeration (recursive, fp64) / LMH programs, masked
lanes, the full-support second pass, the generic resampler (every payload path, partial tiles),
programs over engine results, importance sampling with device-memory data."""
import os
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402

from paper_2010_08454_b200 import Rng, frontend, infer, models, smc  # noqa: E402


def main():
    m = models.HiddenMarkovModel.synthetic(S=20, T=6, seed=1)
    r = smc.SmcRunner(m, 20_000, Rng(1), steps=6, graph=True, hist_steps=[5])
    r.run()
    r.reseed(Rng(2))
    r.run()
    a = smc.SmcRunner(m, 20_000, Rng(3), steps=6, record_ancestors=True)
    a.advance(3)
    snap = a.snapshot()
    b = smc.SmcRunner(m, 20_000, Rng(4), steps=6, record_ancestors=True)
    b.restore(snap)
    b.resume()
    ex = ROOT / "examples"
    for name in ("binomial", "enumerate_geometric", "linear_regression", "linefitting"):
        cm = frontend.compile_program((ex / f"{name}.cup").read_text())
        if cm.engine == "importance":
            infer.run_importance(cm, 50_000, Rng(5))
        elif cm.engine == "enumerate":
            infer.run_enumeration(cm)
        else:
            infer.run_lmh(cm, 50, Rng(6), chains=64)
    os.environ["CUPPL_DSL_LANES"] = "8"  # masked lane form
    cm = frontend.compile_program((ex / "linefitting.cup").read_text())
    infer.run_importance(cm, 50_000, Rng(7), return_traces=True)
    del os.environ["CUPPL_DSL_LANES"]
    from paper_2010_08454_b200 import program, resample

    g = torch.Generator(device="cuda").manual_seed(0)
    for n in (1, 2049, 70_001):
        lw = torch.randn(n, device="cuda", generator=g)
        for pay in (None, torch.arange(n, dtype=torch.int32, device="cuda"),
                    torch.randn((n, 3), device="cuda", generator=g),
                    torch.zeros((n, 5), dtype=torch.uint8, device="cuda"),
                    torch.randn((n, 16), device="cuda", generator=g)):
            resample.systematic(lw, pay, Rng(8), 1, ancestors=True)
    program.run_program("m <- function() { k <- sample(uniform-discrete(0, 3)); k }; p <- enumerate(m, 10); "
                        "dist-var(p)", Rng(9))
    big = models.LinearRegression.synthetic(n_points=5000)
    infer.run_importance(big, 100_000, Rng(10))
    torch.cuda.synchronize()
    print("sanitize_extra done")


if __name__ == "__main__":
    main()
