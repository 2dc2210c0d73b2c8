#!/bin/bash
# End-of-round evidence on one B200 (run through gpurun from the repo root):
#   tools/round_profiles.sh r02
# writes gpurun_out/<tag>/: pytest_gpu.txt, smoke.txt, bench_configs.jsonl.txt,
# bench_ref.json, launches_c2.csv, full_c2.ncu-rep (+ .json / line summaries).
tag=${1:-rXX}
o=gpurun_out/$tag
mkdir -p $o
timeout 1500 python -m pytest tests -m gpu -q > $o/pytest_gpu.txt 2>&1
tail -1 $o/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $o/smoke.txt 2>&1
tail -1 $o/smoke.txt
: > $o/bench_configs.jsonl.txt
timeout 900 python bench.py 2>> $o/bench.err | tail -1 >> $o/bench_configs.jsonl.txt
for c in c1 c3 c4 c5; do
  timeout 900 python bench.py --config $c --no-cpu-baseline 2>> $o/bench.err | tail -1 >> $o/bench_configs.jsonl.txt
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 \
  --master-port 29517 bench.py --gpus 1 --no-cpu-baseline 2>> $o/bench.err | tail -1 >> $o/bench_configs.jsonl.txt
timeout 1200 python bench.py --impl reference --steps 5 --warmup 3 2>> $o/bench.err | tail -1 > $o/bench_ref.json
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $o/launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none \
  -k regex:"k_forward|k_backward_index|k_prepare" -s 9 -c 3 -o $o/full_c2 \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $o/ncu_full.log 2>&1
echo done
