cd $GRAFT_REPO_ROOT
nproc; free -g | head -2
python -m pytest tests/test_gpu_headline.py tests/test_gpu_reference_suite.py tests/test_cli_persist.py tests/test_gpu_properties.py -m gpu -q -s -x -p no:cacheprovider > gpurun_out/batch1.log 2>&1; echo rc=$?
grep -E "rel-L2|reference suite|passed|failed|FAILED|Error" gpurun_out/batch1.log | head -60
