"""Throughput of CuPPL-compiled models vs the hand-written kernels (same model and data)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2010_08454_b200 import Rng, frontend, infer, models  # noqa: E402

LINREG = """
model <- function() {
  a <- sample(normal(0, 10));
  b <- sample(normal(0, 10));
  factor(reduce(function(acc, i) { acc + dist-score(normal(a * xs[i] + b, 1), ys[i]) }, 0.0,
                repeat(function(i) { i }, length(xs))));
  [a, b]
};
importance(model, 1000000)
"""
FIG1 = """
poly <- function(c, x) {
  reduce(function(p, j) { p * x + c[length(c) - 1 - j] }, 0.0, repeat(function(j) { j }, length(c)))
};
distance <- function(c) {
  reduce(function(acc, i) { acc + pow(ys[i] - poly(c, xs[i]), 2) }, 0.0, repeat(function(i) { i }, length(xs)))
};
model <- function() {
  n <- sample(uniform-discrete(2, 5));
  line <- repeat(function(i) { sample(normal(0, 10)) }, n);
  factor(-distance(line));
  line
};
importance(model, 100000)
"""


def rate(launcher, n, reps=3):
    launcher.launch(0, n, Rng(0).key)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(reps):
        launcher.launch(0, n, Rng(k).key)
    e1.record()
    torch.cuda.synchronize()
    return n * reps / (e0.elapsed_time(e1) / 1e3)


def main():
    dev = torch.device("cuda", 0)
    lr = models.LinearRegression.synthetic(n_points=1000)
    poly = models.PolyRegression.synthetic()
    for name, src, model, n in (("linreg D=1000", LINREG, lr, 200_000_000), ("fig1 D=20", FIG1, poly, 2_000_000_000)):
        t0 = time.time()
        m = frontend.compile_program(src, data={"xs": model.xs, "ys": model.ys})
        dl = frontend.DslLauncher(m, dev)
        tc = time.time() - t0
        r_dsl = rate(dl, n)
        r_hand = rate(infer.IsLauncher(model, dev), n)
        print(f"{name}: compiled {r_dsl:.4g} particles/s, hand-written {r_hand:.4g} ({r_dsl / r_hand:.2f}x), "
              f"compile+load {tc:.2f} s")


if __name__ == "__main__":
    main()
