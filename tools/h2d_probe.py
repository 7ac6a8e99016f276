import os, time, torch, torch.distributed as dist
r = int(os.environ["LOCAL_RANK"]); torch.cuda.set_device(r)
dist.init_process_group("nccl", device_id=torch.device("cuda", r))
x = torch.empty(48 * 2**20, dtype=torch.uint8).pin_memory(); y = torch.empty_like(x, device="cuda")
for _ in range(3): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); dist.barrier()
t = time.perf_counter()
for _ in range(40): y.copy_(x, non_blocking=True)
torch.cuda.synchronize(); dt = time.perf_counter() - t
print(f"rank {r} H2D GB/s {40 * x.numel() / dt / 1e9:.1f}", flush=True)
dist.destroy_process_group()
