cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
timeout 300 python tools/fused_probe.py float64 16 > gpurun_out/probe16.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_fused -s 2 -c 2 -o gpurun_out/fused_r2a python tools/fused_probe.py float64 16 > gpurun_out/ncu_fused.log 2>&1
echo rc=$?
tail -3 gpurun_out/ncu_fused.log
