cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/smi.txt
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -rf --durations=25 > gpurun_out/gputests.log 2>&1; echo tests rc=$?
tail -40 gpurun_out/gputests.log
timeout 300 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json | head -c 3000
BTTB_FUSED=1 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-variants --no-e2e > gpurun_out/bench_fused.json 2> gpurun_out/bench_fused.err; echo fused rc=$?
head -c 600 gpurun_out/bench_fused.json
