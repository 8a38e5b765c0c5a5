#!/bin/bash
# A/B tooling: a built copy of a git revision (default HEAD) under prevtree/ (git-ignored, travels to
# the GPU box with the snapshot), so that an A/B runs both versions' own Python bindings and libraries.
REV=${1:-HEAD}
rm -rf prevtree && mkdir prevtree && git archive "$REV" | tar -x -C prevtree
cd prevtree && python -m paper_2504_11651_b200.build > /dev/null && echo "prevtree = $(git rev-parse --short $REV) built"
