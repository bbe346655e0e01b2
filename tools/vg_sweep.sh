# TMA vertex-gather variants (MGPBD_VG_TMA=1) across tile / CTA / ring sizes: pass rate via mgpbd_pass_burst.
# usage: bash tools/vg_sweep.sh "FLAGS" ... -> gpurun_out/vg_sweep.txt
for F in "$@"; do
  MGPBD_EXTRA_NVCC_FLAGS="$F" python paper_2505_13390_b200/build.py --force > gpurun_out/build.log 2>&1 || { echo "build '$F' failed" >> gpurun_out/vg_sweep.txt; continue; }
  echo "== '$F'" >> gpurun_out/vg_sweep.txt
  python tools/pass_env.py "" "MGPBD_VG_TMA=1" >> gpurun_out/vg_sweep.txt 2>&1
done
