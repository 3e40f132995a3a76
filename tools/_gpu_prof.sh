cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
bash tools/profile_round.sh r2b > gpurun_out/prof_r2b.log 2>&1; echo prof rc=$?
ls gpurun_out/r2b | wc -l
