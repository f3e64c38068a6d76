# parity suite + C2/C4 bench with and without programmatic dependent launch
O=gpurun_out
md5sum paper_2407_20474_b200/libfz.so > $O/pdl_md5.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/pdl_tests.log 2>&1; echo "rc=$?" >> $O/pdl_tests.log
for k in 1 2; do
FZ_PDL=0 timeout 300 python bench.py --steps 200 --no-cpu --no-e2e --no-count > $O/pdl_off_$k.json 2>&1
timeout 300 python bench.py --steps 200 --no-cpu --no-e2e --no-count > $O/pdl_on_$k.json 2>&1
done
