O=gpurun_out
timeout 700 python tools/parity_stress.py 40000 20000 600 > $O/r02x_stress_default.log 2>&1; echo "rc=$?" >> $O/r02x_stress_default.log
FZ_ROW_BETA=16 FZ_SLICES_PER_WARP=2 timeout 400 python tools/parity_stress.py 60000 20000 300 > $O/r02x_stress_cost.log 2>&1; echo "rc=$?" >> $O/r02x_stress_cost.log
FZ_ROW_BETA=0 timeout 400 python tools/parity_stress.py 80000 20000 300 > $O/r02x_stress_rows.log 2>&1; echo "rc=$?" >> $O/r02x_stress_rows.log
