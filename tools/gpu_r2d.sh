# K8 wait-before-flush + K1 pre-reduction: parity, all-variant timings, RED counts
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "full_size or small_configs or edge_cases or eigen or many_tiles" > gpurun_out/d_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/d_tests.txt
for c in st27_128 fem_knn_4M spin_22; do
  timeout 600 python bench.py --config $c --no-per-config --all-variants --no-cpu-baseline --steps 200 > gpurun_out/d_var_$c.json 2> gpurun_out/d_var_$c.err; echo "var $c rc=$?"
done
for nv in 0 1; do
  SYMM_K1_PREREDUCE=$((1-nv)) timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed_op_global_red.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_atomic --csv python tools/run_once.py st27_128 atomic > gpurun_out/d_k1_naive$nv.csv 2>&1; echo "ncu k1 naive=$nv rc=$?"
done
