#!/bin/bash
# One gpurun call: GPU tests, the bench line, a step launch list and one --set full capture
# of the step's three kernels (each ncu pass only after the same command exited 0 without ncu).
# Usage: bash profiles/gpu_round.sh TAG [tests|notests]
TAG=${1:-x}; MODE=${2:-tests}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/$TAG.smi 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/$TAG.build.log 2>&1 || { echo BUILD FAIL; tail -30 $O/$TAG.build.log; exit 1; }
if [ "$MODE" = tests ]; then
  timeout 1500 python -m pytest tests -m gpu -x -q > $O/$TAG.pytest.log 2>&1; echo "pytest rc=$?"; tail -5 $O/$TAG.pytest.log
fi
timeout 900 python bench.py > $O/$TAG.bench.json 2> $O/$TAG.bench.err; rc=$?; echo "bench rc=$rc"; tail -c 600 $O/$TAG.bench.json
[ $rc = 0 ] || { tail -30 $O/$TAG.bench.err; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file $O/$TAG.launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra > $O/$TAG.ncu1.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_forward|k_backward_pipe|k_march' \
  --launch-skip 6 -c 3 -o $O/$TAG.full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra > $O/$TAG.ncu2.log 2>&1; echo "ncu full rc=$?"
ls -la $O | tail -20
