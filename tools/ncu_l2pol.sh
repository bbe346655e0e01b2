# L2 residency of the level-0 pass streams under MGPBD_L2POL variants: ncu (no cache flush between kernels) on
# the pass burst of block1.67M fp32.  usage: bash tools/ncu_l2pol.sh 0 1 ... -> gpurun_out/ncu_l2pol_<v>.csv
for V in "$@"; do
  MGPBD_EXTRA_NVCC_FLAGS="-DMGPBD_L2POL=$V" python paper_2505_13390_b200/build.py --force > gpurun_out/build.log 2>&1 || { echo "build $V failed"; continue; }
  timeout 900 ncu --cache-control none --clock-control none -k regex:"k_mf_(vgather|rows)" --launch-skip 800 --launch-count 8 \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read.sum \
    --csv --log-file gpurun_out/ncu_l2pol_$V.csv python - <<'PY' > gpurun_out/ncu_l2pol_$V.log 2>&1
import sys
sys.path.insert(0, ".")
from paper_2505_13390_b200 import mgpbd, scenes
sc = scenes.make("block1.67M")
ctx = mgpbd.Context.from_scene(sc, precision=1)
ctx.step(sc.dt, 2)
print(ctx.pass_burst(400))
PY
done
