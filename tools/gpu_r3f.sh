#!/bin/bash
# Final check of HEAD: GPU tests, smoke, the default bench line and the reference arm
mkdir -p gpurun_out/fin
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin/gputests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/fin/gputests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin/smoke.txt 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/fin/bench_default.json 2> gpurun_out/fin/bench_default.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/fin/bench_reference.json 2> gpurun_out/fin/bench_reference.err; echo "ref rc=$?"
tail -c 600 gpurun_out/fin/bench_reference.json
