import os, sys, torch, torch.distributed as dist
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
dist.init_process_group("gloo", rank=rank, world_size=world)
torch.cuda.set_device(0)
x = torch.arange(4, device="cuda", dtype=torch.int64) + 10 * rank
y = torch.empty_like(x)
for name, fn in (("all_to_all_single", lambda: dist.all_to_all_single(y, x)),
                 ("all_reduce", lambda: dist.all_reduce(x.clone())),
                 ("all_gather", lambda: dist.all_gather([torch.empty_like(x) for _ in range(world)], x))):
    try:
        fn(); torch.cuda.synchronize()
        if rank == 0: print(name, "ok", y.tolist() if name == "all_to_all_single" else "")
    except Exception as e:
        if rank == 0: print(name, "FAILED:", str(e)[:120])
dist.barrier(); dist.destroy_process_group()
