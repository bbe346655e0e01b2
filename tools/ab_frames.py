"""A/B frame timing on a hierarchy that does not depend on the build (GPU box).

The bench's window runs on the hierarchy of a lazy re-setup whose input state carries the rounding of every kernel
before it, so two builds can time different hierarchies (level-1 size varies by a few %, ~1 ms/frame).  Here the
only setup is frame 0's, on the seeded initial state (bit-identical across builds); re-setups are off
(setup_interval 1000, resetup_on_indef 0), so every variant times the same hierarchy A.

  python tools/ab_frames.py [--config block1.67M] [--frames 8] "" "MGPBD_X=1" ...
"""
import argparse
import os
import subprocess
import sys

CHILD = r'''
import os, sys, statistics
sys.path.insert(0, ".")
from paper_2505_13390_b200 import mgpbd, scenes
sc = scenes.make(os.environ["AB_CONFIG"])
ctx = mgpbd.Context.from_scene(sc, precision=1, setup_interval=1000, resetup_on_indef=0)
ms = []
rs = int(os.environ["AB_RESETUP"])
for f in range(rs + 3 + int(os.environ["AB_FRAMES"])):
    if rs and f == rs:
        ctx.setup_hierarchy()   # hierarchy B (deterministic for one build: env variants compare on the same B)
    ctx.step(sc.dt, sc.n_iters)
    if f >= rs + 3:
        ms.append(ctx.stats().ms_frame)
st = ctx.stats()
print(f"median {statistics.median(ms):.3f} ms/frame  min {min(ms):.3f}  levels {[st.n[l] for l in range(st.n_levels)]}", flush=True)
'''


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="block1.67M")
    ap.add_argument("--frames", type=int, default=8)
    ap.add_argument("--resetup-at", type=int, default=0,
                    help="re-setup before this frame (B-type hierarchy; identical across env variants of one build, "
                         "not across builds)")
    ap.add_argument("variants", nargs="*")
    a = ap.parse_args()
    for var in a.variants or [""]:
        env = dict(os.environ, AB_CONFIG=a.config, AB_FRAMES=str(a.frames), AB_RESETUP=str(a.resetup_at))
        for kv in var.split():
            k, v = kv.split("=", 1)
            env[k] = v
        r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=900)
        print(repr(var), r.stdout.strip() or r.stderr[-400:], flush=True)


if __name__ == "__main__":
    main()
