#!/bin/bash
# One gpurun call: GPU tests, smoke, bench, ncu launch list + one full capture.
# usage: gpurun --timeout 1500 -- bash tools/gpu_round.sh [tag] [what...]
set -u
cd "${GRAFT_REPO_ROOT:-$(dirname "$0")/..}"
TAG=${1:-r1}; shift || true
WHAT=${*:-"tests smoke bench ncu"}
OUT=gpurun_out/$TAG
mkdir -p "$OUT"
nvidia-smi -L > "$OUT/gpu.txt" 2>&1
for w in $WHAT; do
  case $w in
    tests) timeout 900 python -m pytest tests -x -q -m gpu -p no:cacheprovider > "$OUT/pytest_gpu.txt" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.txt";;
    quick) timeout 600 python -m pytest tests -x -q -m gpu -p no:cacheprovider -k "not c2_full and not large_tree" > "$OUT/pytest_gpu.txt" 2>&1; echo "pytest rc=$?" >> "$OUT/pytest_gpu.txt";;
    smoke) timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > "$OUT/smoke.txt" 2>&1; echo "smoke rc=$?" >> "$OUT/smoke.txt";;
    bench) timeout 600 python bench.py > "$OUT/bench.json" 2> "$OUT/bench.err"; echo "bench rc=$?" >> "$OUT/bench.err";;
    bench_simple) RS_SIMPLE_QUERY=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > "$OUT/bench_simple.json" 2>> "$OUT/bench.err";;
    bench_binary) RS_BINARY_FAST=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > "$OUT/bench_binary.json" 2>> "$OUT/bench.err";;
    bench_quad) RS_TRAV_LANES=4 timeout 600 python bench.py --no-cpu-baseline --no-e2e > "$OUT/bench_quad.json" 2>> "$OUT/bench.err";;
    bench_presort) timeout 600 python bench.py --presort --no-cpu-baseline --no-e2e > "$OUT/bench_presort.json" 2>> "$OUT/bench.err";
                   RS_TRAV_LANES=4 timeout 600 python bench.py --presort --no-cpu-baseline --no-e2e > "$OUT/bench_presort_quad.json" 2>> "$OUT/bench.err";
                   RS_BINARY_FAST=1 timeout 600 python bench.py --presort --no-cpu-baseline --no-e2e > "$OUT/bench_presort_binary.json" 2>> "$OUT/bench.err";;
    bench_presort_simple) RS_SIMPLE_QUERY=1 RS_BINARY_FAST=1 timeout 600 python bench.py --presort --no-cpu-baseline --no-e2e > "$OUT/bench_presort_simple.json" 2>> "$OUT/bench.err";
                   RS_SIMPLE_QUERY=1 RS_BINARY_FAST=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > "$OUT/bench_simple.json" 2>> "$OUT/bench.err";;
    bench_buffer) RS_FAST_PATH=buffer timeout 600 python bench.py --no-cpu-baseline --no-e2e > "$OUT/bench_buffer.json" 2>> "$OUT/bench.err";;
    bench_sbin) RS_SORTED_BINARY=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > "$OUT/bench_sbin.json" 2>> "$OUT/bench.err";;
    bench_mb) for mb in ${RS_MBS:-6}; do for c in ${RS_CFGS:-c2 c3 c4}; do RS_LIB=paper_2209_02878_b200/lib/libraysurf_b200_mb$mb.so timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 > "$OUT/bench_${c}_mb$mb.json" 2>> "$OUT/bench.err"; done; done;;
    bench_mb_old) for mb in 8 10; do RS_LIB=paper_2209_02878_b200/lib/libraysurf_b200_mb$mb.so timeout 600 python bench.py --no-cpu-baseline --no-e2e > "$OUT/bench_mb$mb.json" 2>> "$OUT/bench.err"; done;;
    bench_nograph) RS_NO_GRAPH=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > "$OUT/bench_nograph.json" 2>> "$OUT/bench.err";;
    benchq) timeout 600 python bench.py --no-cpu-baseline > "$OUT/bench.json" 2>> "$OUT/bench.err";;
    stats) timeout 300 python tools/stats.py c2 > "$OUT/stats_c2.json" 2>&1;;
    ncuq) timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_query|k_trav|k_exact|k_bin' -s 6 -c 5 \
        -o "$OUT/query" python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/ncu_full.log" 2>&1;;
    bench_c3) timeout 600 python bench.py --config c3 --no-cpu-baseline --steps 20 > "$OUT/bench_c3.json" 2>> "$OUT/bench.err";;
    bench_var) for v in ${RS_VARS:-bin tile}; do for c in ${RS_CFGS:-c2 c3 c4 c5}; do RS_TRAV=$v timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 > "$OUT/bench_${c}_$v.json" 2>> "$OUT/bench.err"; done; done;;
    bench_area) for ar in ${RS_AREAS:-16 32 48 96}; do for c in ${RS_CFGS:-c2 c4 c5}; do RS_TILE_AREA=$ar timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 > "$OUT/bench_${c}_a$ar.json" 2>> "$OUT/bench.err"; done; done;;
    bench_env) # RS_ENVS="A=1,B=2 A=3" : one bench per env set (commas -> spaces)
      for ev in ${RS_ENVS:-RS_NONE=1}; do for c in ${RS_CFGS:-c2}; do tag=$(echo "$ev" | sed 's|paper_2209_02878_b200/lib/||g' | tr ',=/' '_-_'); env $(echo "$ev" | tr ',' ' ') timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 > "$OUT/bench_${c}_$tag.json" 2>> "$OUT/bench.err"; done; done;;
    ncuk) # full capture of kernels matching RS_NCU_K (regex) in one step of config RS_NCU_CFG
      timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${RS_NCU_K:-k_bin}" -s ${RS_NCU_SKIP:-10} -c ${RS_NCU_C:-3} \
        -o "$OUT/k_${RS_NCU_CFG:-c2}" python bench.py --config ${RS_NCU_CFG:-c2} --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/ncu_k.log" 2>&1;;
    ncut) timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_trav' -s 3 -c 1 \
        -o "$OUT/trav_${RS_NCU_CFG:-c2}" python bench.py --config ${RS_NCU_CFG:-c2} --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/ncu_trav.log" 2>&1;;
    e2e_env) for ev in ${RS_ENVS:-RS_NONE=1}; do for c in ${RS_CFGS:-c2}; do tag=$(echo "$ev" | sed 's|paper_2209_02878_b200/lib/||g' | tr ',=/' '_-_'); env $(echo "$ev" | tr ',' ' ') timeout 300 python bench.py --config $c --no-cpu-baseline --steps 20 > "$OUT/e2e_${c}_$tag.json" 2>> "$OUT/bench.err"; done; done;;
    klist) # per-kernel serialized times for each env set in RS_ENVS (or default), config RS_CFGS
      for ev in ${RS_ENVS:-RS_NONE=1}; do for c in ${RS_CFGS:-c2}; do tag=$(echo "$ev" | sed 's|paper_2209_02878_b200/lib/||g' | tr ',=/' '_-_');
        env $(echo "$ev" | tr ',' ' ') timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
          --log-file "$OUT/kl_${c}_$tag.csv" python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>> "$OUT/bench.err";
        python tools/launch_table.py "$OUT/kl_${c}_$tag.csv" 18 > "$OUT/kl_${c}_$tag.txt"; done; done;;
    ab) # interleaved A/B of libraries RS_LIBS (names under lib/, default "base ''") on RS_CFGS
      for rep in 1 2; do for l in ${RS_LIBS:-base cur}; do for c in ${RS_CFGS:-c2 c4 c5}; do
        if [ "$l" = cur ]; then lib=paper_2209_02878_b200/lib/libraysurf_b200.so; else lib=paper_2209_02878_b200/lib/libraysurf_b200_$l.so; fi
        RS_LIB=$lib timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps ${RS_AB_STEPS:-30} > "$OUT/ab_${c}_${l}_$rep.json" 2>> "$OUT/bench.err"
      done; done; done;;
    abenv) # interleaved A/B of env sets RS_ENVS ("A=1,B=2 A=3"; commas -> spaces) on RS_CFGS
      for rep in 1 2 3; do for ev in ${RS_ENVS:-RS_NONE=1}; do for c in ${RS_CFGS:-c2}; do
        tag=$(echo "$ev" | tr ',=/' '_-_')
        env $(echo "$ev" | tr ',' ' ') timeout 300 python bench.py --config $c --no-cpu-baseline --no-e2e --steps ${RS_AB_STEPS:-100} > "$OUT/ab_${c}_${tag}_$rep.json" 2>> "$OUT/bench.err"
      done; done; done;;
    sanitize) for tool in memcheck synccheck racecheck; do
        arg=""; [ $tool = racecheck ] && arg=small
        timeout 1200 compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize.py $arg > "$OUT/sanitize_$tool.txt" 2>&1
        echo "rc=$?" >> "$OUT/sanitize_$tool.txt"; done;;
    traffic) for c in ${RS_CFGS:-c2 c3 c4 c5}; do
        timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
          --clock-control none --csv --log-file "$OUT/traffic_$c.csv" python bench.py --config $c --steps 2 \
          --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/traffic_$c.log" 2>&1
        python tools/traffic.py "$OUT/traffic_$c.csv" $c --out "$OUT/traffic_$c.json" >> "$OUT/traffic_$c.log" 2>&1; done;;
    fullhot) for c in ${RS_CFGS:-c2}; do
        timeout 900 ncu --set full --clock-control none --import-source on -k regex:${RS_HOT:-k_trav_tile} -s 3 -c 1 \
          -o "$OUT/full_$c" python bench.py --config $c --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/full_$c.log" 2>&1; done;;
    bench_all) for c in c2 c3 c4 c5; do timeout 900 python bench.py --config $c --steps ${RS_ALL_STEPS:-10} > "$OUT/bench_$c.json" 2>> "$OUT/bench.err"; done;;
    ncu)
      timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
        --log-file "$OUT/launches.csv" python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/ncu_bench.log" 2>&1
      timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_|onesweep' -s 40 -c 20 \
        -o "$OUT/full" python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > "$OUT/ncu_full.log" 2>&1;;
  esac
done
ls -la "$OUT"
