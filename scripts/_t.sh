python -m pytest tests/test_free_gpu.py -q 2>&1 | tail -2
python -m pytest tests/test_dist_gpu.py -q 2>&1 | tail -2
python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 scripts/probe_dist.py 2>&1 | grep -v "^W\|OMP\|\*\*\*\*\|NCCL version" | head -12
