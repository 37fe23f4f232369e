# A/B: spill targets of short-run tiles read from the block's global copy before
# the stage wait (default build) vs from the staged block (base.so), and two
# consumer/gather warp shapes; parity of the default build first
mkdir -p gpurun_out; : > gpurun_out/r3a_summary.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "not full_size" > gpurun_out/r3a_tests.txt 2>&1; tail -3 gpurun_out/r3a_tests.txt >> gpurun_out/r3a_summary.txt
run() {  # label lib variant config
  SYMM_LIB=$2 timeout 300 python bench.py --config $4 --no-per-config --no-cpu-baseline --variant $3 --steps 300 > gpurun_out/r3a.json 2> gpurun_out/r3a.err
  python -c "import json;d=json.load(open('gpurun_out/r3a.json'));print('$4 $3 $1',round(d['ms_per_step'],4),round(d['roofline']['frac'],3),d['clocks']['sm_mhz'],d.get('parity_sampled_relinf'))" >> gpurun_out/r3a_summary.txt 2>&1 || tail -2 gpurun_out/r3a.err >> gpurun_out/r3a_summary.txt
}
for c in fem_knn_4M spin_22 st27_128; do
  for v in tiled_atomic tiled_colored; do
    run "tgt_global (default)" "" $v $c
    run "base (tgt from block)" libvariants/base.so $v $c
    [ $v = tiled_atomic ] && run "4x6 consumers + 6 gather" libvariants/g6gw6.so $v $c
    [ $v = tiled_atomic ] && run "3x9 consumers + 3 gather" libvariants/g3x9.so $v $c
  done
done
cat gpurun_out/r3a_summary.txt
