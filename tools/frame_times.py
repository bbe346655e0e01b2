"""Per-frame device times of a config through the C-ABI with CUDA graphs (no profiling), for A/B runs.

  python tools/frame_times.py --config block1.67M --frames 12 [--precision fp32]
Prints one summary line: median / min of the frames without a setup, setups, indefinite events.
"""
import argparse
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2505_13390_b200 import mgpbd, scenes  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="block1.67M")
    ap.add_argument("--frames", type=int, default=12)
    ap.add_argument("--precision", default="fp32")
    ap.add_argument("--tag", default="")
    a = ap.parse_args()
    sc = scenes.make(a.config)
    ctx = mgpbd.Context.from_scene(sc, precision=1 if a.precision == "fp32" else 0)
    plain, setups, ev, trace = [], 0, 0, []
    for f in range(a.frames):
        ctx.step(sc.dt, sc.n_iters)
        s = ctx.stats()
        ev += s.indefinite_events
        trace.append(f"{s.ms_frame:.1f}{'S' if s.setup_ran else ''}{'!' + str(s.indefinite_events) if s.indefinite_events else ''}")
        if s.setup_ran:
            setups += 1
        elif f > 0:
            plain.append(s.ms_frame)
    print(f"{a.tag} {a.config} {a.precision}: frames w/o setup median {statistics.median(plain):.2f} ms, "
          f"min {min(plain):.2f} ms (n={len(plain)}), setups {setups}, indefinite events {ev} | {' '.join(trace)}",
          flush=True)


if __name__ == "__main__":
    main()
