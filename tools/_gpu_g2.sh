cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_properties.py tests/test_gpu_reference_suite.py -m gpu -q -p no:cacheprovider -x > gpurun_out/t2.log 2>&1; echo tests rc=$?
tail -5 gpurun_out/t2.log
bash tools/sanitize.sh
