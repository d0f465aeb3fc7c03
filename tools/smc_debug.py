"""Debug one SMC step on the GPU against the oracle: tile prefixes, ancestors."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import core  # noqa: E402
from paper_2010_08454_b200 import models, smc  # noqa: E402

KEY = 0x9E0160293A33AAF7


def main(n=100_000, S=50, steps=2):
    n, S, steps = int(n), int(S), int(steps)
    m = models.HiddenMarkovModel.synthetic(S=S, T=steps, seed=1)
    r = smc.SmcRunner(m, n, KEY, record_ancestors=True, steps=steps)
    r.init()
    r.step(0)
    torch.cuda.synchronize()
    rk = r.ranks[0]
    ws = rk.ws.cpu().numpy()
    nt = (n + 4095) // 4096
    al = lambda v: (v + 255) & ~255
    off = al(nt * 8) + al(16) + al(nt * 16)
    tp = ws[off:off + nt * 8].view(np.uint64)
    print("n_tiles", nt, "tile_prefix[:6]", tp[:6], "T", r.gathered[0].cpu().numpy()[:, 0])
    for t in range(1, steps):
        r.step(t)
    torch.cuda.synchronize()
    r._snapshot_ancestors()
    ref = core.smc_run(m, n, KEY, steps=steps, record_ancestors=True)
    print("T gpu", r.gathered[:, 0, 0].cpu().numpy().view(np.uint64), "T ref", ref["T"])
    for t in range(steps - 1):
        anc = r.ancestors[t][0].cpu().numpy().astype(np.int64)
        ra = ref["ancestors"][t].astype(np.int64)
        bad = np.nonzero(anc != ra)[0]
        print("step", t, "mismatches", len(bad))
        if len(bad):
            print("  first bad", bad[:10], anc[bad[:10]], ra[bad[:10]])
            b = bad[0]
            print("  around", anc[max(0, b - 3):b + 4], ra[max(0, b - 3):b + 4])
            break


if __name__ == "__main__":
    main(*sys.argv[1:])
