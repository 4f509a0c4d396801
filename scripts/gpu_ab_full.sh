#!/bin/bash
# every GPU test on the new build, then same-box A/B of libpi_base.so (A) vs the new libpi.so (B)
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
AB_CFGS="${AB_CFGS:-c4:1 c3:1 c2:1}" bash scripts/gpu_ab.sh
