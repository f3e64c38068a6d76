O=gpurun_out; T=${1:-r02r}
for i in 1 2; do
(cd ab/r1 && timeout 300 python tools/quick_time.py C2 C2h C3t2 > ../../$O/${T}_r1_$i.log 2>&1)
(cd ab/varA && timeout 300 python tools/quick_time.py C2 C2h C3t2 T95 > ../../$O/${T}_varA_$i.log 2>&1)
timeout 300 python tools/quick_time.py C2 C2h C3t2 T95 C3t3 > $O/${T}_head_$i.log 2>&1
done
timeout 900 python -m pytest tests -m gpu -x -q > $O/${T}_tests.log 2>&1; echo "rc=$?" >> $O/${T}_tests.log
