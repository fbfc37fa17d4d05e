set -u
OUT=gpurun_out/r2y; mkdir -p $OUT
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_host.py -x -q -m gpu -p no:cacheprovider -k "bary or scene or soup or layered or c2_full or knobs or variants or chunked or unpermute or sort_rays or edge or lean or sweep or adversarial or garbage" > $OUT/pytest.txt 2>&1; echo "rc=$?" >> $OUT/pytest.txt
for c in c3 c2; do timeout 600 python bench.py --config $c --no-cpu-baseline > $OUT/bench_$c.json 2>> $OUT/bench.err; done
