# Build-time sweep of the level-0 matrix-free pass, measured with mgpbd_pass_burst on block1.67M (GPU box).
# usage: bash tools/pass_sweep.sh "FLAGS_A" "FLAGS_B" ...   -> gpurun_out/pass_sweep.txt
for F in "$@"; do
  MGPBD_EXTRA_NVCC_FLAGS="$F" python paper_2505_13390_b200/build.py --force > gpurun_out/build.log 2>&1 || { echo "build '$F' failed" >> gpurun_out/pass_sweep.txt; continue; }
  FL="$F" timeout 300 python - >> gpurun_out/pass_sweep.txt 2>>gpurun_out/err.log <<'PY'
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
print(repr(os.environ["FL"]), " | ".join(out), flush=True)
PY
done
