python tools/pass_probe.py --algo cc --scale 27 --uniform --reps 2 > gpurun_out/c4_pass.txt 2>&1
ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/c4_pass_launches.csv python tools/pass_probe.py --algo cc --scale 27 --uniform --reps 1 > /dev/null 2>&1
cat gpurun_out/c4_pass.txt
python tools/launch_table.py gpurun_out/c4_pass_launches.csv --full 2>&1 | head -60
