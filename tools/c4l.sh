for v in ${VARIANTS:-base a0}; do
SERAPH_LIB=$PWD/variants/libseraph_$v.so ncu --profile-from-start off --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/c4l_$v.csv python tools/pass_probe.py --algo cc --scale 27 --uniform --reps 1 > gpurun_out/c4l_$v.txt 2>&1
python tools/launch_table.py gpurun_out/c4l_$v.csv --full 2>&1 | head -40
done
