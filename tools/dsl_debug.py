"""Debug a compiled program: constant data read back from the module, a few particles vs the
fp64 interpreter."""
import importlib.util
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402
from cuda.bindings import driver as cu  # noqa: E402

from oracle.dsl_eval import Interpreter  # noqa: E402
from paper_2010_08454_b200 import Rng, frontend, infer  # noqa: E402

spec = importlib.util.spec_from_file_location("t", str(Path(__file__).resolve().parent.parent / "tests/test_frontend.py"))
t = importlib.util.module_from_spec(spec)
spec.loader.exec_module(t)
for name in sys.argv[1:] or ["FIG1", "LINREG"]:
    src = getattr(t, name)
    m = frontend.compile_program(src)
    post = infer.run_importance(m, 64, Rng(3), return_traces=True)
    h = __import__("hashlib").sha256(m.cuda.encode() + m.data.tobytes() + repr(frontend._lanes_to_try(m)).encode()).hexdigest()
    mod = frontend._MODULES[h][0]
    err, dptr, size = cu.cuModuleGetGlobal(mod, b"DC")
    buf = np.zeros(size // 4, dtype=np.float32)
    cu.cuMemcpyDtoH(buf.ctypes.data, dptr, size)
    print(name, "data", m.data, "module DC", buf, "match", np.array_equal(buf, m.data))
    lw = post.traces["log_weight"].cpu().numpy()
    draws = post.traces["draws"].cpu().numpy()
    it = Interpreter(src)
    for i in range(4):
        print("  ", lw[i], it.run(draws[i])[0], draws[i])
