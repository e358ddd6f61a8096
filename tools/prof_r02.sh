# Round-2 profiling pass (run under gpurun; every ncu command after the plain run exited 0).
# Reports are summarised ON the box (details + raw CSV pages) and then removed:
# gpurun copies back at most 64 MiB.
set -x
mkdir -p gpurun_out
summ() {  # $1 = report base name
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed > gpurun_out/$1_raw.csv 2>/dev/null
  python tools/ncu_details.py gpurun_out/$1.ncu-rep gpurun_out/$1_summary.csv
  ncu -i gpurun_out/$1.ncu-rep --page source --csv --kernel-name regex:"$2" --launch-skip 0 --launch-count 1 > gpurun_out/$1_source.csv 2>/dev/null
  rm -f gpurun_out/$1.ncu-rep
}
./tools/micro/tf32_peak > gpurun_out/tf32_peak.json 2>&1; echo tf32_rc=$?
python tools/legprof.py c4 1 3 > gpurun_out/c4_legprof.txt 2>&1; echo c4plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_down_staged|k_up_staged|k_adots|k_update|k_conv_tc|k_conv_rows" -c 40 -o gpurun_out/c4_full -f python tools/legprof.py c4 1 3 > gpurun_out/ncu_c4.log 2>&1; echo ncu_c4_rc=$?
summ c4_full k_down_staged
python tools/c0prof.py 148 1 > gpurun_out/c0_plain.txt 2>&1; echo c0plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_down_staged|k_up_staged|k_down_lean|k_up_stream|k_adots|k_update|k_coarse_reg" --launch-skip 300 -c 14 -o gpurun_out/c0_full -f python tools/c0prof.py 148 1 > gpurun_out/ncu_c0.log 2>&1; echo ncu_c0_rc=$?
summ c0_full k_adots
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --also "" --no-cpu --groups 1 > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch_rc=$?
du -sh gpurun_out
