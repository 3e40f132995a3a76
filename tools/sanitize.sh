#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over the operator's kernels
# (VERDICT r1 item 6): C1, C2 and a two-layer C4 block (2048^2 FFTs: the TMA
# row / column stages, mbarrier pipelines and the mirrored row passes), default
# path and the fused layer pipeline (BTTB_PIPE=1).  Logs -> gpurun_out/sanitize/.
cd ${GRAFT_REPO_ROOT:-.}
OUT=gpurun_out/sanitize
mkdir -p $OUT
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  for case in "C1 float64" "C2 float64" "C4L float64" "C4L float32"; do
    set -- $case
    for pipe in 0 1; do
      [ "$pipe" = 1 ] && [ "$1" != C4L ] && continue
      log=$OUT/${tool}_$1_$2_pipe$pipe.log
      BTTB_PIPE=$pipe timeout 900 $CS --tool $tool --error-exitcode 99 --print-limit 50 \
        python tools/sanitize_case.py $1 $2 > $log 2>&1
      echo "$tool $1 $2 pipe=$pipe rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|forward' $log | tr '\n' ' ')"
    done
  done
done
