# launch list of the C2 step with the memo build split into separate kernels (FZ_FUSE_MEMO=0)
O=gpurun_out
FZ_FUSE_MEMO=0 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -s 30 -c 60 --csv --log-file $O/split_c2.csv python bench.py --steps 20 --warmup 10 --no-e2e --no-cpu --no-count > $O/split.log 2>&1
for g in 16 32 64 148; do FZ_K1_GRID=$g timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k1 -s 5 -c 5 --csv --log-file $O/grid_$g.csv python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu --no-count > /dev/null 2>&1; done
