#!/bin/bash
# Fast GPU iteration: build, the render parity tests, a short bench line (no CPU legs) and
# the step launch list.  Optional: NCU=<kernel regex> adds one --set full capture of it.
# Usage: bash profiles/gpu_iter.sh TAG ["pytest -k expr or test files"]
TAG=${1:-it}; TESTS=${2:-"tests/test_gpu_parity.py tests/test_gpu_render_variants.py tests/test_gpu_configs.py"}
O=gpurun_out; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/$TAG.build.log 2>&1 || { echo BUILD FAIL; tail -30 $O/$TAG.build.log; exit 1; }
if [ "$TESTS" != none ]; then
  timeout 900 python -m pytest $TESTS -m gpu -x -q > $O/$TAG.pytest.log 2>&1; echo "pytest rc=$?"; tail -4 $O/$TAG.pytest.log
fi
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extra ${BENCH_ARGS} > $O/$TAG.bench.json 2> $O/$TAG.bench.err; rc=$?
echo "bench rc=$rc"; python - <<PY
import json
d=json.load(open("$O/$TAG.bench.json"))
r=d["roofline"]
print("ms/step", round(d["ms_per_step"],3), "value %.4g"%d["value"], "fwd_call", round(r["fwd_call_ms"],3), "bwd", round(r["bwd_ms"],3), "clk", d["clocks"]["sm_mhz"])
PY
[ $rc = 0 ] || { tail -30 $O/$TAG.bench.err; exit 1; }
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 140 --csv --log-file $O/$TAG.launches.csv \
  python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-extra ${BENCH_ARGS} > $O/$TAG.ncu1.log 2>&1; echo "ncu launches rc=$?"
python profiles/launch_list.py $O/$TAG.launches.csv 3 | tail -20
if [ -n "$NCU" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$NCU" --launch-skip ${NCU_SKIP:-3} -c ${NCU_C:-1} \
    -o $O/$TAG.full -f python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra ${BENCH_ARGS} > $O/$TAG.ncu2.log 2>&1; echo "ncu full rc=$?"
fi
