#!/bin/bash
# Large-block factor check on the GPU box: parity on the 12^3/16^3 goldens,
# Table-3 timings, and a launch list of the 2D config-2 step.
# usage: tools/gpu_check_lg.sh TAG
set -u
TAG=${1:-lg}
mkdir -p gpurun_out
python -m pytest tests/test_gpu_parity.py -m gpu -q -k "b16 or b1644" > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
python -m paper_1707_07598_b200.table3bench --geometry table3 --repeats 5 --out gpurun_out/${TAG}_t3 > gpurun_out/${TAG}_t3.log 2>&1
echo "table3 rc=$?"; tail -8 gpurun_out/${TAG}_t3.log
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_cfg2.csv \
    python bench.py --config 2 --steps 1 --warmup 3 > gpurun_out/${TAG}_cfg2_ncu.log 2>&1
echo "cfg2 ncu rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}_t3.csv \
    python -m paper_1707_07598_b200.table3bench --geometry table3 --repeats 1 --out gpurun_out/${TAG}_t3ncu > gpurun_out/${TAG}_t3_ncu.log 2>&1
echo "t3 ncu rc=$?"
