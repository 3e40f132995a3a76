cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
BTTB_FUSED_STATS=1 timeout 300 python tools/fused_probe.py float64 128 2>&1 | tail -6
BTTB_FUSED_STATS=1 timeout 300 python tools/fused_probe.py float32 128 2>&1 | tail -6
