"""Pipe-rate calibration on the GPU box: FFMA2, FFMA, Philox, MUFU (csrc/calib_kernels.cu)."""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

from paper_2010_08454_b200 import _native as N  # noqa: E402


def main():
    L = N.lib()
    dev = torch.device("cuda", 0)
    sink = torch.zeros(256, device=dev)
    sm = torch.cuda.get_device_properties(dev).multi_processor_count
    out = {"sm_count": sm}
    for kind, name, per_iter in [(0, "ffma2_flops", 512.0), (1, "ffma_flops", 256.0),
                                 (2, "philox_blocks", 1.0), (3, "mufu_ops", 64.0),
                                 (4, "lr_fadd2_ffma2_particle_points", 128.0),
                                 (5, "lr_3ffma2_particle_points", 128.0),
                                 (6, "lr_scalar_particle_points", 128.0),
                                 (7, "fadd2_lane_ops", 256.0), (8, "fadd_lane_ops", 256.0)]:
        for blocks_per_sm in (4, 8, 16):
            blocks, iters = sm * blocks_per_sm, 2000 if kind != 2 else 200
            for _ in range(2):
                N.check(L.cuppl_calibrate(kind, blocks, iters, N.ptr(sink), N.stream_ptr()))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            N.check(L.cuppl_calibrate(kind, blocks, iters, N.ptr(sink), N.stream_ptr()))
            e1.record()
            torch.cuda.synchronize()
            s = e0.elapsed_time(e1) / 1e3
            rate = blocks * 256 * iters * per_iter / s
            out[f"{name}@{blocks_per_sm}cta"] = rate
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
