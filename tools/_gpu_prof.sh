cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 1800 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_headline.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
bash tools/profile_round.sh r2d > gpurun_out/prof_r2d.log 2>&1; echo prof rc=$?
