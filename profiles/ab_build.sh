#!/bin/bash
# Build the current sources as a named side-by-side variant libsvr_b200.<name>.so for A/B
# timing on one GPU box (SVR_LIB_VARIANT=<name> python bench.py ...).
set -e
NAME=$1
cd /root/repo
python -c "from paper_2305_13220_b200 import build; build.build(force=True)"
cp paper_2305_13220_b200/libsvr_b200.so paper_2305_13220_b200/libsvr_b200.$NAME.so
echo built libsvr_b200.$NAME.so
