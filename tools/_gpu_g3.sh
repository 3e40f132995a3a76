cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python -m pytest tests/test_gpu_guards.py tests/test_gpu_bench_multirank.py tests/test_gpu_properties.py tests/test_gpu_reference_suite.py -m gpu -q -p no:cacheprovider -rf -s > gpurun_out/t3.log 2>&1; echo tests rc=$?
grep -E "passed|failed|worst|guard|Error|error" gpurun_out/t3.log | tail -40
