#!/bin/bash
# GPU parity tests of the default build, then the A/B bench of every variant (scripts/ab.sh).
mkdir -p gpurun_out
TAG=${1:-abt}
{
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
} > gpurun_out/${TAG}_tests.log 2>&1
cat gpurun_out/${TAG}_tests.log
bash scripts/ab.sh ${TAG}
