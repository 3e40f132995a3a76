cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
python tools/step_probe.py float64 128 2>&1 | tail -2
python tools/step_probe.py float32 128 2>&1 | tail -2
bash tools/profile_round.sh r2a > gpurun_out/prof_r2a.log 2>&1; echo prof rc=$?
ls gpurun_out/r2a
python tools/step_probe.py float64 128 2>&1 | tail -2
