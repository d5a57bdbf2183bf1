# A/B of block-sweep variants against the default build: lower-triangle inverse
# (tri), 9 / 10 / 12 warps per CTA with 3 / 4 / 4 / 6 solver warps
cd $GRAFT_REPO_ROOT
for v in "" tri w9 w10 w12 w12s6; do
  PHI_VARIANT=$v timeout 300 python tools/ab_variant.py c2 3 >> gpurun_out/ab.log 2>&1
  PHI_VARIANT=$v timeout 300 python tools/ab_variant.py c3 2 1 >> gpurun_out/ab.log 2>&1
done
PHI_VARIANT="" timeout 300 python tools/ab_variant.py c2 3 >> gpurun_out/ab.log 2>&1
