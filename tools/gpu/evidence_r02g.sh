# round-2 final evidence refresh (usage: bash tools/gpu/evidence_r02g.sh TAG): GPU parity suite, bench lines (N = 1; C4
# headline; 2 ranks sharing the GPU over gloo; reference arm), ncu launch lists and full captures (CSV exported on
# the box), per-config timings, Table 1.  (compute-sanitizer is closed on this pool: see profiles/r02e_sanitizers.md)
T=${1:-r02g}
O=gpurun_out
md5sum paper_2407_20474_b200/libfz.so > $O/${T}_md5.txt
nvidia-smi --query-gpu=name,clocks.max.sm,clocks.sm --format=csv > $O/${T}_smi.txt 2>&1
exp() {
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  ncu -i $O/$1.ncu-rep --page source --csv --print-source sass > $O/$1_source.csv 2>/dev/null
  gzip -f $O/$1_source.csv
  rm -f $O/$1.ncu-rep
}
timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
timeout 600 python bench.py > $O/${T}_bench.json 2> $O/${T}_bench.err
timeout 300 python bench.py --config C4 --steps 20 --no-cpu > $O/${T}_bench_c4.json 2> $O/${T}_bench_c4.err
timeout 600 python bench.py --gpus 2 --steps 20 > $O/${T}_bench_2rank.json 2> $O/${T}_bench_2rank.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $O/${T}_bench_reference.json 2> $O/${T}_bench_reference.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 60 --csv --log-file $O/${T}_launches_c2.csv python bench.py --steps 20 --warmup 10 --no-e2e --no-cpu --no-count > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 12 -c 12 --csv --log-file $O/${T}_launches_c4.csv python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu --no-count > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'k1_memo|k5_walk|k4_plan' -s 6 -c 3 -o $O/${T}_c2 python tools/prof_one.py C2 4 > /dev/null 2>&1; exp ${T}_c2
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'k5_runs' -s 1 -c 1 -o $O/${T}_c4 python tools/prof_one.py C4 2 > /dev/null 2>&1; exp ${T}_c4
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'k5_walk' -s 1 -c 1 -o $O/${T}_c3t3 python tools/prof_one.py C3t3 2 > /dev/null 2>&1; exp ${T}_c3t3
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'k5_walk' -s 1 -c 1 -o $O/${T}_t95 python tools/prof_one.py T95 2 > /dev/null 2>&1; exp ${T}_t95
timeout 300 python tools/quick_time.py C2 C2h C2c C3t2 C3t3 C3t4 C4 C4t2 T1 T95 T94 T63 T74 > $O/${T}_quick_time.log 2>&1
timeout 300 python tools/table1_bench.py > $O/${T}_table1.log 2>&1
