#!/bin/bash
# A/B matrix of env switches / build variants on the C4 bench (run under gpurun).
#   bash tools/variants.sh "label1|ENV=1 ENV2=0" "label2|BTTB_LIB_PATH=build/x/libbttb_sm100.so" ...
# Prints one line per variant: ms/step fp64, fwd, tra, fp32 ms/step.
mkdir -p gpurun_out/var
for spec in "$@"; do
  label="${spec%%|*}"; envs="${spec#*|}"
  env $envs timeout 300 python bench.py --steps ${STEPS:-30} --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var/$label.log 2>&1
  python - "$label" << 'PY'
import json, sys
lab = sys.argv[1]
try:
    d = json.loads(open(f"gpurun_out/var/{lab}.log").read().strip().splitlines()[-1])
    print(f"{lab:24s} f64 {d['ms_per_step']:.3f} ms (fwd {d['fwd_ms']:.3f} tra {d['tra_ms']:.3f}) "
          f"f32 {d['variants']['f32']['ms_per_step']:.3f} ms  L={d['config']['fft_shape']} clk={d['clocks']['sm_mhz']}")
except Exception as e:
    print(lab, "FAILED", e, open(f"gpurun_out/var/{lab}.log").read()[-400:])
PY
done
