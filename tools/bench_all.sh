#!/bin/bash
# Every config's bench line and reference arm (round-2 record under profiles/).
O=gpurun_out
for c in 1 2 3 4 5; do
  extra=""; [ $c = 5 ] && extra="--no-cpu-baseline"
  python bench.py --config $c $extra > $O/r02_bench_config$c.json 2> $O/r02_bench_config$c.err
  python bench.py --config $c --impl reference > $O/r02_reference_config$c.json 2> $O/r02_reference_config$c.err
done
python bench.py --config 5 --sharding row --no-cpu-baseline > $O/r02_bench_config5_row1.json 2> $O/r02_bench_config5_row1.err
python tools/lambda_sweep.py > $O/r02_lambda_sweep.json 2> $O/ls.err
ls -la $O/r02_*
