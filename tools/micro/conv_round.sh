python tools/convacc.py 4 128; python tools/convacc.py 5 128
ncu --kernel-name regex:k_conv_tc --clock-control none --metrics gpu__time_duration.sum -c 16 --csv --log-file gpurun_out/sk3.csv python tools/convbench.py 4 128 8 > /dev/null 2>&1
python tools/convbench.py 5 512 2 2>&1 | head -2
