# Round-2 LAST profiling pass (after the k_adots index change), c0 at the default batch (888 replicas =
# 3 column groups of 296): ncu --set full of one group's kernels, the launch list, the traffic per class.
set -x
mkdir -p gpurun_out
summ() {  # $1 = report base name
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum > gpurun_out/$1_raw.csv 2>/dev/null
  python tools/ncu_details.py gpurun_out/$1.ncu-rep gpurun_out/$1_summary.csv
  rm -f gpurun_out/$1.ncu-rep
}
python tools/c0prof.py 296 1 > gpurun_out/c0_plain.txt 2>&1; echo c0plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_down_row|k_up_row|k_adots|k_update|k_coarse_reg|k_finalize|k_restart" --launch-skip 300 -c 16 -o gpurun_out/r02f_c0_full -f python tools/c0prof.py 296 1 > gpurun_out/ncu_c0.log 2>&1; echo ncu_c0_rc=$?
summ r02f_c0_full
python tools/ncu_traffic.py gpurun_out/r02f_c0_full_raw.csv "ncu --set full, tools/c0prof.py 296 1 (one c0 column group of 296, launches 300-315), round 2 final (profiles/r02f_c0_full_raw.csv)" > gpurun_out/ncu_traffic.log 2>&1; cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json 2>/dev/null
python bench.py --steps 2 --warmup 3 --also "" --no-cpu --groups 1 --replicas 296 > gpurun_out/launch_plain.json 2>&1; echo launch_plain_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02f_c0_launches.csv python bench.py --steps 2 --warmup 3 --also "" --no-cpu --groups 1 --replicas 296 > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch_rc=$?
python tools/launches.py gpurun_out/r02f_c0_launches.csv > gpurun_out/r02f_c0_launch_shares.txt 2>&1
