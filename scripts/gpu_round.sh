#!/bin/bash
# One GPU iteration: smoke + GPU parity tests, A/B bench of lib/variants (scripts/ab.sh), ncu capture.
TAG=${1:-round}
mkdir -p gpurun_out
{
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
} > gpurun_out/${TAG}_tests.log 2>&1
cat gpurun_out/${TAG}_tests.log
CONFIGS=${CONFIGS:-llama8b_block llama70b_block} bash scripts/ab.sh ${TAG}
bash scripts/gpu_prof_only.sh ${TAG}
