set -u
OUT=gpurun_out/r2final; mkdir -p $OUT
nvidia-smi -L > $OUT/gpu.txt
timeout 1500 python -m pytest tests -q -m gpu -p no:cacheprovider > $OUT/pytest_gpu.txt 2>&1; echo "rc=$?" >> $OUT/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.txt 2>&1; echo "smoke rc=$?" >> $OUT/smoke.txt
timeout 900 python bench.py > $OUT/bench_c2.json 2>> $OUT/bench.err
for c in c3 c4 c5; do timeout 900 python bench.py --config $c --steps 50 > $OUT/bench_$c.json 2>> $OUT/bench.err; done
timeout 900 python bench.py --impl reference --steps 10 --warmup 3 > $OUT/ref_c2.json 2>> $OUT/bench.err
