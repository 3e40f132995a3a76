cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-variants > gpurun_out/b_e2e.json 2> gpurun_out/b_e2e.err
python -c "import json; d=json.load(open('gpurun_out/b_e2e.json')); print(d['ms_per_step'], d['e2e'])"
timeout 600 python -m pytest tests/test_gpu_properties.py tests/test_gpu_parity.py tests/test_gpu_cgls.py -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
