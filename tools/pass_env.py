"""Level-0 pass rate (mgpbd_pass_burst) on block1.67M under environment-switch variants (no rebuild).

  python tools/pass_env.py "" "MGPBD_NO_VG_TMA=1" ...
"""
import os
import subprocess
import sys

CHILD = r'''
import os, sys
sys.path.insert(0, ".")
from paper_2505_13390_b200 import mgpbd, scenes
sc = scenes.make(os.environ.get("SWEEP_CONFIG", "block1.67M"))
out = []
for prec in (1, 0):
    ctx = mgpbd.Context.from_scene(sc, precision=prec)
    ctx.step(sc.dt, 2)
    ms, by = ctx.pass_burst(200)
    out.append(f"fp{'32' if prec else '64'} {by / 200 / 1e6:.1f} MB/pass {ms / 200 * 1e3:.2f} us/pass {by / ms / 1e6:.0f} GB/s")
    ctx.close()
print(" | ".join(out), flush=True)
'''

for var in sys.argv[1:] or [""]:
    env = dict(os.environ)
    for kv in var.split():
        k, v = kv.split("=", 1)
        env[k] = v
    r = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True, timeout=600)
    print(repr(var), r.stdout.strip() or r.stderr[-300:], flush=True)
