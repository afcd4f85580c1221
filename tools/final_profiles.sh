# Round-end evidence on one B200 (about 25 minutes): GPU tests, both bench arms, the ncu launch
# list and one --set full capture per headline kernel, the status log and the FP64 operand probes.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-n-level --no-scaling-samples > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bloch_wave_kernel -c 1 -o gpurun_out/r2_cfg2 python tools/prof_step.py cfg2 --steps 20000 --no-warm > gpurun_out/ncu_cfg2.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_step_kernel -c 1 -o gpurun_out/r2_cfg4 python tools/prof_step.py cfg4 --no-warm > gpurun_out/ncu_cfg4.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:dense_step_kernel -c 1 -o gpurun_out/r2_cfg3 python tools/prof_step.py cfg3 --no-warm > gpurun_out/ncu_cfg3.log 2>&1
bash tools/status.sh > gpurun_out/status.log 2>&1
python tools/fp64_peaks.py > gpurun_out/fp64_peaks.log 2>&1
(python tools/nlevel_rate.py; python tools/nlevel_rate.py --stepper rk4 --levels 2 3 4 5 6 7 8) > gpurun_out/nlevel_rates.log 2>&1
python tools/parity_report.py > gpurun_out/parity.log 2>&1
