mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/bench.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-n-level --no-scaling-samples > gpurun_out/ncu_launch.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bloch_wave_kernel -c 1 -o gpurun_out/r2_cfg2 python tools/prof_step.py cfg2 --steps 20000 --no-warm > gpurun_out/ncu_cfg2.log 2>&1
