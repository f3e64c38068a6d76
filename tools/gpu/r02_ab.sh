# same-box A/B: round-1 library (ab/r1) vs HEAD
O=gpurun_out; T=${1:-r02n}
for i in 1 2; do
(cd ab/r1 && timeout 300 python tools/quick_time.py C3t2 C3t3 C2h C2 C4 T95 T94 > ../../$O/${T}_r1_$i.log 2>&1)
timeout 300 python tools/quick_time.py C3t2 C3t3 C2h C2 C4 T95 T94 > $O/${T}_head_$i.log 2>&1
done
