# round-2 checkpoint: GPU tests, default bench (headline + per_config), force-dist, ncu launch list
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/c_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/c_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c_tests.txt
timeout 900 python bench.py > gpurun_out/c_bench.json 2> gpurun_out/c_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/c_bench.err
timeout 600 python bench.py --force-dist --config st27_128 --steps 100 --no-per-config > gpurun_out/c_fd.json 2> gpurun_out/c_fd.err; echo "force-dist rc=$?"; tail -3 gpurun_out/c_fd.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c_launches_lap3d_512.csv python bench.py --steps 3 --warmup 3 --no-per-config --no-cpu-baseline --soak-ms 0 > gpurun_out/c_ncu.log 2>&1; echo "ncu rc=$?"
