# A/B: block inverse stored as its lower triangle (PHI_BLK_TRI, _lib_tri) vs the default build
cd $GRAFT_REPO_ROOT
for rep in 1 2; do
for v in "" tri; do
  PHI_VARIANT=$v python tools/ab_variant.py c2 3 >> gpurun_out/ab_tri.log 2>&1
  PHI_VARIANT=$v python tools/ab_variant.py c3 2 1 >> gpurun_out/ab_tri.log 2>&1
done; done
PHI_VARIANT=tri timeout 900 python -m pytest tests/test_gpu_fast.py tests/test_gpu_determinism.py -x -q > gpurun_out/ab_tri_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/ab_tri_pytest.log
