# round-1 evidence pass: launch lists, ncu full captures (exported to CSV on the box), multi-rank bench checks
set -x
O=gpurun_out
exp() {  # export an ncu report to CSV pages and drop the binary (gpurun_out/ must stay < 64 MiB)
  ncu -i $O/$1.ncu-rep --page raw --csv > $O/$1_raw.csv 2>/dev/null
  ncu -i $O/$1.ncu-rep --page details --csv > $O/$1_details.csv 2>/dev/null
  ncu -i $O/$1.ncu-rep --page source --csv --print-source sass > $O/$1_source.csv 2>/dev/null
  gzip -f $O/$1_source.csv
  rm -f $O/$1.ncu-rep
}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 60 --csv --log-file $O/r01b_launches_c2.csv python bench.py --steps 20 --warmup 10 --no-e2e --no-cpu --no-count > $O/ncu_l.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 9 -c 9 --csv --log-file $O/r01b_launches_c4.csv python bench.py --config C4 --steps 3 --warmup 3 --no-e2e --no-cpu > $O/ncu_l4.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'k1_memo|k5_walk|k4_plan' -s 6 -c 3 -o $O/r01b_c2 python tools/prof_one.py C2 4 > $O/ncu_f.log 2>&1; exp r01b_c2
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'k5_walk' -s 1 -c 1 -o $O/r01b_c4 python tools/prof_one.py C4 2 > $O/ncu_f4.log 2>&1; exp r01b_c4
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'k5_walk' -s 1 -c 1 -o $O/r01b_c3t3 python tools/prof_one.py C3t3 2 > $O/ncu_f3.log 2>&1; exp r01b_c3t3
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 20 --warmup 3 > $O/tr2_c2.json 2> $O/tr2_c2.err
FZ_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 20 --warmup 3 > $O/tr2g_c2.json 2> $O/tr2g_c2.err
FZ_BENCH_BACKEND=gloo timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --config C4 --steps 5 --warmup 3 > $O/tr2g_c4.json 2> $O/tr2g_c4.err
timeout 200 python bench.py --steps 50 --no-cpu --no-count > $O/b1.json 2> $O/b1.err
timeout 200 python tools/quick_time.py C3t2 C3t3 C3t4 C2h C4 > $O/qt.log 2>&1
ls -la $O
