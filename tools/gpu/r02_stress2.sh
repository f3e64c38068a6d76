O=gpurun_out
timeout 800 python tools/parity_stress.py 100000 40000 720 > $O/r02z_stress.log 2>&1; echo "rc=$?" >> $O/r02z_stress.log
