#!/bin/bash
# Re-entry evidence of HEAD: GPU tests, then the round evidence script.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/x_tests.txt 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/x_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/x_smoke.txt 2>&1; echo "smoke rc=$?"
bash tools/gpu_round_evidence.sh
ls gpurun_out/ev
