#!/bin/bash
# 2 GPUs: C2 e2e with and without the windowed column upload, interleaved, build phase timings
O=gpurun_out
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
for i in 1 2; do
  CHROMA_BUILD_TIMING=1 timeout 300 $TR --nproc-per-node 2 --master-port 2983$i bench.py --gpus 2 > $O/ab_win_$i.json 2> $O/ab_win_$i.err
  CHROMA_NO_WINDOW=1 CHROMA_BUILD_TIMING=1 timeout 300 $TR --nproc-per-node 2 --master-port 2984$i bench.py --gpus 2 > $O/ab_full_$i.json 2> $O/ab_full_$i.err
done
for f in $O/ab_*.json; do echo $f; python -c "import json; d=json.load(open('$f')); print(d['ms_per_step'], d['value'], d['e2e']['value'])"; done
grep -h "col h2d" $O/ab_win_1.err | tail -4; echo ---; grep -h "col h2d" $O/ab_full_1.err | tail -4
