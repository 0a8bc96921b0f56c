"""World-1 NCCL check of bench.strip_vcycle_timing (the N>1 bench V-cycle path) on one GPU."""
import os, sys, json
sys.path.insert(0, os.getcwd())
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
import torch, torch.distributed as dist
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1)
import bench
print(json.dumps(bench.strip_vcycle_timing(0, 1)))
dist.destroy_process_group()
