# Mid-size reference goldens through the CUDA path, both schedules
# (diff against the reference's per-pair decision log).
for c in ${CASES:-imq3d_n32768 imq3d_n32768_leaf8 imq3d_n16384_leaf16 c2_exp2d_n65536}; do
  for sch in reference wavefront; do
    IFMM_TRACE=/tmp/tr_${c}_$sch.txt timeout 900 python tools/diff_mid.py $c $sch > gpurun_out/mid_$c.$sch.log 2>&1
  done
done
tail -n 40 gpurun_out/mid_*.log
