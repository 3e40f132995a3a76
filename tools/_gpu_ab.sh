cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_cgls.py tests/test_gpu_generic.py tests/test_gpu_variants.py tests/test_gpu_headline.py tests/test_gpu_entries.py tests/test_gpu_properties.py -m gpu -q -p no:cacheprovider -x 2>&1 | tail -2
STEPS=20 bash tools/variants.sh "u1|X=1" "u2|X=1" "u3|X=1"
python bench.py --config C5 --dtype f32 --cgls 10 --steps 10 --no-cpu-baseline 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('C5 cgls', d['ms_per_step'])"
