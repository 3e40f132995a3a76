cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_generic.py tests/test_gpu_reference_suite.py -m gpu -q -p no:cacheprovider -rf -x > gpurun_out/gen.log 2>&1; echo tests rc=$?
tail -30 gpurun_out/gen.log
