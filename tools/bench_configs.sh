#!/bin/bash
# bench lines for the other BASELINE configs (json into gpurun_out/cfg<N>.json)
mkdir -p gpurun_out
for c in 3 5; do
  python bench.py --config $c --steps 10 --warmup 3 --no-cpu-baseline --no-gn --no-table3 > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.err
  echo "config $c rc=$?"
done
for c in 1 2; do
  python bench.py --config $c --steps 10 --warmup 3 > gpurun_out/cfg$c.json 2> gpurun_out/cfg$c.err
  echo "config $c rc=$?"
done
