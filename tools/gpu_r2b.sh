mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/b_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/b_tests.txt
timeout 900 python bench.py > gpurun_out/b_bench.json 2> gpurun_out/b_bench.err; echo "bench rc=$?"; tail -3 gpurun_out/b_bench.err
timeout 300 python bench.py --gpus 2 > gpurun_out/b_g2.json 2>&1; echo "gpus2 rc=$?"; cat gpurun_out/b_g2.json | tail -2
timeout 600 python bench.py --force-dist --config st27_128 --steps 100 > gpurun_out/b_fd.json 2> gpurun_out/b_fd.err; echo "force-dist rc=$?"; tail -3 gpurun_out/b_fd.err
