#!/bin/bash
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_dist.py -q -x -p no:cacheprovider 2>&1 | tail -3
timeout 600 python bench.py --config cfg5 --steps 1 --warmup 1 2>&1 | tail -1
