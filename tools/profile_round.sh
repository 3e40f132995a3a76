#!/bin/bash
# Round measurement set (run under gpurun from the repo root):
#   bench (default), reference arm, one-step ncu launch list (recipe metric and
#   warm-cache DRAM bytes), and one full ncu capture of the top kernels.
# Outputs go to gpurun_out/$1/.
set -x
R=${1:-r1}
OUT=gpurun_out/$R
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/smi.txt
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python bench.py --impl reference > $OUT/bench_ref.json 2> $OUT/bench_ref.err
python bench.py --config C5 --dtype f32 --cgls 10 --steps 10 > $OUT/cgls_c5.json 2> $OUT/cgls_c5.err
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file $OUT/launches_cgls_c5.csv python bench.py --config C5 --dtype f32 --cgls 10 --profile-step > $OUT/ncu_cgls.log 2>&1
for DT in f64 f32; do
  python bench.py --dtype $DT --profile-step --no-cpu-baseline --no-variants --no-e2e > $OUT/plain_$DT.log 2>&1 && \
  ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv \
      --log-file $OUT/launches_$DT.csv python bench.py --dtype $DT --profile-step --no-cpu-baseline --no-variants --no-e2e > $OUT/ncu1_$DT.log 2>&1
  ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum \
      --cache-control none --clock-control none --csv \
      --log-file $OUT/traffic_$DT.csv python bench.py --dtype $DT --profile-step --no-cpu-baseline --no-variants --no-e2e > $OUT/ncu2_$DT.log 2>&1
done
ncu --profile-from-start off --set full --import-source on --cache-control none --clock-control none \
    -k regex:"k_col_fwd|k_col_tra|k_row_r2c_t2d|k_row_c2r_t2d|k_row_c2r_mirror" -c 6 \
    -o $OUT/full_f64 python bench.py --profile-step --no-cpu-baseline --no-variants --no-e2e > $OUT/ncu3.log 2>&1
ncu -i $OUT/full_f64.ncu-rep --page raw --csv > $OUT/full_f64_raw.csv 2>/dev/null
ncu -i $OUT/full_f64.ncu-rep --page details --csv > $OUT/full_f64_details.csv 2>/dev/null
ncu --profile-from-start off --set full --cache-control none --clock-control none \
    -k regex:"k_row_r2c_t2d|k_row_c2r_mirror" -c 4 -o $OUT/full_f32 python bench.py --dtype f32 --profile-step --no-cpu-baseline --no-variants --no-e2e > $OUT/ncu5.log 2>&1
ncu -i $OUT/full_f32.ncu-rep --page raw --csv > $OUT/full_f32_raw.csv 2>/dev/null
rm -f $OUT/full_f32.ncu-rep
ncu --profile-from-start off --set full --import-source on --cache-control none --clock-control none \
    -k regex:"k_col" -c 4 -o $OUT/full_c5 python bench.py --config C5 --dtype f32 --cgls 10 --profile-step > $OUT/ncu4.log 2>&1
ncu -i $OUT/full_c5.ncu-rep --page raw --csv > $OUT/full_c5_raw.csv 2>/dev/null
rm -f $OUT/full_f64.ncu-rep $OUT/full_c5.ncu-rep
echo done
