cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=15 > gpurun_out/gputests.log 2>&1; echo tests rc=$?
tail -25 gpurun_out/gputests.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
python -c "
import json; d=json.load(open('gpurun_out/bench.json'))
print(d['ms_per_step'], d['fwd_ms'], d['tra_ms'], d['roofline']['frac'], d['e2e']['value'], d['clocks'], d['variants']['f32']['ms_per_step'], d.get('parity'))"
