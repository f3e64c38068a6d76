O=gpurun_out; T=${1:-r02k}
timeout 1500 python bench.py --study f4 > $O/${T}_f4_study.jsonl 2> $O/${T}_f4_study.err
