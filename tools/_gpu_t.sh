cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_integration_stub.py tests/test_gpu_reference_suite.py -m gpu -q -p no:cacheprovider -rf 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()"
