"""Generate golden fixtures from the reference implementation (run in the build container).

Imports the reference's own `cuppl.rng` and `cuppl.values` from /root/reference (read-only)
and records their outputs, so tests can pin this package's mirrors without the reference
present (it does not exist on the GPU box).

    python tests/golden/make_golden.py   ->  tests/golden/refrng.json
"""

import json
import sys
from pathlib import Path

REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))

from cuppl.rng import Rng  # noqa: E402
from cuppl import values  # noqa: E402

out = {"source": "cuppl.rng / cuppl.values from /root/reference/pkg/src", "streams": [], "splits": []}
for seed, stream in [(0, 0), (1, 0), (1, 1), (42, 7), (2**63 + 5, 3), (123456789, 0)]:
    r = Rng(seed, stream)
    rec = {"seed": seed, "stream": stream, "key": r.key,
           "next_u64": [r.next_u64() for _ in range(4)]}
    r = Rng(seed, stream)
    rec["uniform"] = [r.uniform() for _ in range(4)]
    r = Rng(seed, stream)
    rec["randint3"] = [r.randint(3) for _ in range(6)]
    r = Rng(seed, stream)
    rec["normal_0_10"] = [r.normal(0.0, 10.0) for _ in range(5)]
    r = Rng(seed, stream)
    rec["beta_2_3"] = [r.beta(2.0, 3.0) for _ in range(3)]
    r = Rng(seed, stream)
    rec["poisson_4"] = [r.poisson(4.0) for _ in range(4)]
    r = Rng(seed, stream)
    rec["exponential_2"] = [r.exponential(2.0) for _ in range(3)]
    out["streams"].append(rec)
    base = Rng(seed, stream)
    out["splits"].append({"seed": seed, "stream": stream,
                          "children": [[i, base.split(i).key] for i in (0, 1, 2, 1000, 10**11)]})

vk = []
for v in [None, True, False, 0, 1, 1.0, -2.5, "s", (1, 2.0), (True, (1,))]:
    vk.append({"value": repr(v), "key": repr(values.value_key(v))})
out["value_key"] = vk
dst = Path(__file__).resolve().parent / "refrng.json"
dst.write_text(json.dumps(out, indent=1))
print(dst)
