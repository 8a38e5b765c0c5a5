#!/bin/bash
# A/B of lib/variants (no tests) + phase profile of the prof.so variant if present.
TAG=${1:-abp}
mkdir -p gpurun_out
if [ -f paper_2504_11651_b200/lib/variants/prof.so ]; then
  for c in ${PCONFIGS:-llama8b_block}; do
    DF11_LIB=paper_2504_11651_b200/lib/variants/prof.so python scripts/phase_profile.py $c 2>&1 | tail -10
  done > gpurun_out/${TAG}_phase.log
  mv paper_2504_11651_b200/lib/variants/prof.so /tmp/prof.so
fi
cat gpurun_out/${TAG}_phase.log 2>/dev/null
CONFIGS=${CONFIGS:-llama8b_block llama70b_block} bash scripts/ab.sh ${TAG}
