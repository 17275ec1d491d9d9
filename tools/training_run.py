"""Measured adaptive training run (the B200 form of the
reference's run_training_sim / speedup_summary, src/adaptive.cpp:34-129):
scene trajectory early-training -> late-training, both candidate kernels
timed on the device per keyframe, selector checkpoints every interval.

  python tools/training_run.py [--iters 7000 --keyframes 8 --interval 1000] [--out profiles/r1_training_run.csv]
"""
import argparse
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2412_17378_b200 import _native as N  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=7000)
    ap.add_argument("--keyframes", type=int, default=8)
    ap.add_argument("--interval", type=int, default=1000)
    ap.add_argument("--n", type=int, default=1_000_000)
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "training_run.csv"))
    a = ap.parse_args()
    p = N.TrainingParams(a.iters, a.keyframes, 1920, 1080, 16, 16, 1000.0, a.n, 42, 0.05, 1.0, 0.02, 0.035, 0.05, 1.0)
    # one run (measured times differ run to run, so the text length is not
    # known up front): a buffer far above 7000 rows x ~80 characters
    cap = max(1 << 20, a.iters * 160)
    need = C.c_size_t(0)
    buf = C.create_string_buffer(cap)
    N.call("bs_host_run_training", C.byref(p), a.interval, buf, cap, C.byref(need))
    if need.value >= cap:
        raise RuntimeError(f"report truncated ({need.value} bytes)")
    text = buf.value.decode()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        f.write(text)
    print([ln for ln in text.splitlines() if ln.startswith("# summary")][0])


if __name__ == "__main__":
    main()
