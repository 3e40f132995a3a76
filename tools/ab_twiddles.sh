# A/B of the TMEM twiddle cache (BTTB_TW_TMEM) under gpurun: parity subset, C4 f64/f32 and C5 benches
cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_headline.py tests/test_gpu_cgls.py tests/test_gpu_reference_suite.py tests/test_gpu_fuzz.py -q -p no:cacheprovider -x > gpurun_out/ab_tests.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/ab_tests.log
for tw in 1 0 1 0; do
  for dt in f64 f32; do
    BTTB_TW_TMEM=$tw timeout 300 python bench.py --dtype $dt --no-variants --no-cpu-baseline --no-e2e > gpurun_out/ab_${dt}_$tw.json 2>/dev/null
    python -c "import json; d=json.load(open('gpurun_out/ab_${dt}_$tw.json')); print('$dt tw=$tw', round(d['ms_per_step'],4), round(d['fwd_ms'],4), round(d['tra_ms'],4), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
  done
  BTTB_TW_TMEM=$tw timeout 300 python bench.py --config C5 --dtype f32 --cgls 10 --steps 10 > gpurun_out/ab_c5_$tw.json 2>/dev/null
  python -c "import json; d=json.load(open('gpurun_out/ab_c5_$tw.json')); print('C5 tw=$tw', round(d['ms_per_step'],4))"
done
