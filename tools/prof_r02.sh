# Round-2 profiling pass (run under gpurun; every ncu command runs after the same
# command exited 0 without ncu).  Reports are summarised ON the box (details +
# raw CSV pages) and removed: gpurun copies back at most 64 MiB.
set -x
mkdir -p gpurun_out
summ() {  # $1 = report base name
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active > gpurun_out/$1_raw.csv 2>/dev/null
  python tools/ncu_details.py gpurun_out/$1.ncu-rep gpurun_out/$1_summary.csv
  rm -f gpurun_out/$1.ncu-rep
}
./tools/micro/tf32_peak > gpurun_out/tf32_peak.json 2>&1; echo tf32_rc=$?
# c0 x 148 (one column group): the bench's per-launch sizes
python tools/c0prof.py 148 1 > gpurun_out/c0_plain.txt 2>&1; echo c0plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_down_staged|k_up_staged|k_down_lean|k_up_stream|k_adots|k_update|k_coarse_reg" --launch-skip 300 -c 14 -o gpurun_out/r02_c0_full -f python tools/c0prof.py 148 1 > gpurun_out/ncu_c0.log 2>&1; echo ncu_c0_rc=$?
summ r02_c0_full
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r02_c0_launches.csv python bench.py --steps 2 --warmup 3 --also "" --no-cpu --groups 1 > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch_rc=$?
# c4: the real config (4096^2, 4 levels, ABL 32, U-Net coarse at 512^2), 3 FGMRES(20) iterations
python tools/legprof.py c4 1 3 > gpurun_out/c4_legprof.txt 2>&1; echo c4plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_down_staged|k_up_staged|k_adots|k_update|k_conv_tc|k_conv_rows" -c 40 -o gpurun_out/r02_c4_full -f python tools/legprof.py c4 1 3 > gpurun_out/ncu_c4.log 2>&1; echo ncu_c4_rc=$?
summ r02_c4_full
# c2: the cluster-resident coarsest GMRES at 128^2 (8 columns)
python tools/debug/coarse_bench.py 512 8 > gpurun_out/cc_plain.txt 2>&1; echo ccplain_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_coarse_cluster" -c 1 -o gpurun_out/r02_c2_coarse_cluster -f python tools/debug/coarse_bench.py 512 8 > gpurun_out/ncu_cc.log 2>&1; echo ncu_cc_rc=$?
summ r02_c2_coarse_cluster
# paper U-Net on tcgen05 (UNetConfig() at 128^2, batch 16)
python tools/debug/paper_layers_tc.py 16 > gpurun_out/paper_layers.txt 2>&1; echo paper_rc=$?
timeout 600 ncu --set full --clock-control none -k regex:"k_conv_tc" -c 12 -o gpurun_out/r02_paper_tc -f python tools/debug/paper_layers_tc.py 16 > gpurun_out/ncu_paper.log 2>&1; echo ncu_paper_rc=$?
summ r02_paper_tc
du -sh gpurun_out
