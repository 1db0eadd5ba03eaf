import os, torch, torch.distributed as dist, torch.multiprocessing as mp
def w(rank):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29611")
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    x = torch.ones(3, device="cuda") * (rank + 1)
    dist.all_reduce(x)
    y = torch.empty(6, device="cuda")
    try:
        dist.all_gather_into_tensor(y, x)
        ag = y.tolist()
    except Exception as e:
        ag = f"ERR {e}"
    print(rank, x.tolist(), ag, flush=True)
    dist.destroy_process_group()
if __name__ == "__main__":
    mp.spawn(w, nprocs=2)
