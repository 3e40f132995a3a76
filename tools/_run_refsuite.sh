cd $GRAFT_REPO_ROOT
python -m pytest tests/test_gpu_reference_suite.py -m gpu -q -s -x > gpurun_out/refsuite.log 2>&1; echo rc=$?
tail -80 gpurun_out/refsuite.log
