# Round-2 (final state, session 4) profiling pass: the c0 kernels after the full-row legs /
# two-CTA coarse solve, the c0 launch list, the c4 legs and Krylov kernels, and
# the two-CTA conv_rows layers.  Every ncu command runs after the same command
# exited 0 without ncu; reports are summarised on the box and removed.
set -x
mkdir -p gpurun_out
summ() {  # $1 = report base name
  ncu -i gpurun_out/$1.ncu-rep --page details --csv > gpurun_out/$1_details.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,launch__grid_size,launch__block_size,launch__registers_per_thread,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__throughput.avg.pct_of_peak_sustained_elapsed,gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum > gpurun_out/$1_raw.csv 2>/dev/null
  python tools/ncu_details.py gpurun_out/$1.ncu-rep gpurun_out/$1_summary.csv
  rm -f gpurun_out/$1.ncu-rep
}
python tools/c0prof.py 148 1 > gpurun_out/c0_plain.txt 2>&1; echo c0plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_down_row|k_up_row|k_adots|k_update|k_coarse_reg|k_finalize|k_restart" --launch-skip 300 -c 16 -o gpurun_out/r02d_c0_full -f python tools/c0prof.py 148 1 > gpurun_out/ncu_c0.log 2>&1; echo ncu_c0_rc=$?
summ r02d_c0_full
python tools/ncu_traffic.py gpurun_out/r02d_c0_full_raw.csv "ncu --set full, tools/c0prof.py 148 1 (c0 x148, launches 300-315), round 2 session 4 final (profiles/r02d_c0_full_raw.csv)" > gpurun_out/ncu_traffic.log 2>&1; cp profiles/ncu_traffic.json gpurun_out/ncu_traffic.json 2>/dev/null
python bench.py --steps 2 --warmup 3 --also "" --no-cpu --groups 1 > gpurun_out/launch_plain.json 2>&1; echo launch_plain_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/r02d_c0_launches.csv python bench.py --steps 2 --warmup 3 --also "" --no-cpu --groups 1 > gpurun_out/ncu_launch.log 2>&1; echo ncu_launch_rc=$?
python tools/launches.py gpurun_out/r02d_c0_launches.csv > gpurun_out/r02d_c0_launch_shares.txt 2>&1
# c4: 4096^2, 4 levels, U-Net coarse at 512^2, 3 FGMRES(20) iterations
python tools/legprof.py c4 1 3 > gpurun_out/c4_legprof.txt 2>&1; echo c4plain_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_down_staged|k_up_staged|k_adots|k_update" -c 24 -o gpurun_out/r02d_c4_full -f python tools/legprof.py c4 1 3 > gpurun_out/ncu_c4.log 2>&1; echo ncu_c4_rc=$?
summ r02d_c4_full
# c2 U-Net forward (L=5, 512^2 x 16): the conv layers' tensor-pipe activity
python tools/convbench.py 5 512 16 > gpurun_out/conv_c2_plain.txt 2>&1; echo conv_rc=$?
timeout 900 ncu --set full --clock-control none -k regex:"k_conv" -c 30 -o gpurun_out/r02d_conv_c2 -f python tools/convbench.py 5 512 16 > gpurun_out/ncu_conv.log 2>&1; echo ncu_conv_rc=$?
summ r02d_conv_c2
du -sh gpurun_out
# paper U-Net (UNetConfig() at 128^2, batch 16): per-layer event times, then ncu of its tcgen05 convs
python tools/debug/paper_layers_tc.py 16 > gpurun_out/r02d_paper_layers.txt 2>&1; echo paper_rc=$?
timeout 600 ncu --set full --clock-control none -k regex:"k_conv_tc" -c 16 -o gpurun_out/r02d_paper_tc -f python tools/debug/paper_layers_tc.py 16 > gpurun_out/ncu_paper.log 2>&1; echo ncu_paper_rc=$?
summ r02d_paper_tc
# the c3 apply per layer (context split, per-slice conv_rows)
python tools/debug/cfg_layers.py c3 64 > gpurun_out/r02d_c3_layers.txt 2>&1; echo c3_rc=$?
