set -x
python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err
echo bench_rc=$?
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --also "" --no-cpu --groups 1 > gpurun_out/ncu_launch.log 2>&1
echo ncu1_rc=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_coarse_reg|k_down_lean|k_up_stream|k_adots|k_update" --launch-skip 300 -c 10 -o gpurun_out/c0_full python tools/c0prof.py 148 1 > gpurun_out/ncu_full.log 2>&1
echo ncu2_rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_up_staged|k_down_staged|k_adots|k_update" -c 12 -o gpurun_out/c4_legs python tools/legprof.py 4096 1 2 > gpurun_out/ncu_c4.log 2>&1
echo ncu3_rc=$?
