cd $GRAFT_REPO_ROOT
export PYTHONDONTWRITEBYTECODE=1
echo "default: $(python tools/step_probe.py float32 128 2>&1 | tail -2 | tr '\n' ' ')"
echo "QUAD=0: $(BTTB_QUAD=0 python tools/step_probe.py float32 128 2>&1 | tail -2 | tr '\n' ' ')"
mkdir -p gpurun_out/f32
ncu --profile-from-start off --set full --cache-control none --clock-control none \
    -k regex:"k_row_r2c_t2d|k_row_c2r_mirror" -c 4 -o gpurun_out/f32/full_f32 python bench.py --dtype f32 --profile-step --no-cpu-baseline --no-variants --no-e2e > gpurun_out/f32/ncu.log 2>&1
ncu -i gpurun_out/f32/full_f32.ncu-rep --page raw --csv > gpurun_out/f32/full_f32_raw.csv 2>/dev/null
rm -f gpurun_out/f32/full_f32.ncu-rep
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/f32/full_f32_raw.csv")))
hdr = rows[0]
keys = ["gpu__time_duration.sum", "l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__average_warp_latency_issue_stalled_barrier", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem"]
for r in rows[2:]:
    print(r[hdr.index("Kernel Name")][:50], {k.split("__")[1][:30]: r[hdr.index(k)] for k in keys if k in hdr})
PY
