set -u
OUT=gpurun_out/r2av; mkdir -p $OUT
for c in c2 c3 c4; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e > $OUT/bench_$c.json 2>> $OUT/bench.err; done
