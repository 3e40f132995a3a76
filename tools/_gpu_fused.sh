cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "c4 or odd or small" -p no:cacheprovider > gpurun_out/fused_parity.log 2>&1; echo parity rc=$?
tail -5 gpurun_out/fused_parity.log
timeout 300 python bench.py --steps 20 --warmup 5 > gpurun_out/fused_bench.log 2>&1; echo bench rc=$?
tail -c 3000 gpurun_out/fused_bench.log
