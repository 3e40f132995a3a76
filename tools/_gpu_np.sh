cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
nproc
python tools/numpy_path_probe.py 2>&1 | tail -4
timeout 900 python -m pytest tests/test_gpu_properties.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
