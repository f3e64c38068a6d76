# GPU parity suite + one full ncu capture of the C4 COUNT walk (exported to CSV here)
O=gpurun_out
md5sum paper_2407_20474_b200/libfz.so > $O/c4p_md5.txt
timeout 900 python -m pytest tests -m gpu -x -q > $O/c4p_tests.log 2>&1; echo "rc=$?" >> $O/c4p_tests.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:'k5_walk' -s 1 -c 1 -o $O/c4p python tools/prof_one.py C4 2 > $O/c4p_ncu.log 2>&1
ncu -i $O/c4p.ncu-rep --page raw --csv > $O/c4p_raw.csv 2>/dev/null
ncu -i $O/c4p.ncu-rep --page source --csv --print-source sass > $O/c4p_source.csv 2>/dev/null; gzip -f $O/c4p_source.csv
rm -f $O/c4p.ncu-rep
