import os, socket, sys
import torch, torch.distributed as dist, torch.multiprocessing as mp
def port():
    s = socket.socket(); s.bind(("127.0.0.1", 0)); p = s.getsockname()[1]; s.close(); return p
def worker(rank, world, prt):
    os.environ["MASTER_ADDR"] = "127.0.0.1"; os.environ["MASTER_PORT"] = str(prt)
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = torch.cuda.Stream()
    for n in (1000, 1 << 20, 3 << 20):
        # 1: plain
        x = torch.full((n,), float(rank + 1), device="cuda")
        dist.all_reduce(x); torch.cuda.synchronize()
        ok1 = bool((x == 3).all())
        # 2: side stream after event, value produced by a kernel right before
        y = torch.zeros(n, device="cuda"); y += (rank + 1); ev = torch.cuda.Event(); ev.record()
        comm.wait_event(ev)
        with torch.cuda.stream(comm):
            dist.all_reduce(y)
        torch.cuda.current_stream().wait_stream(comm); torch.cuda.synchronize()
        ok2 = bool((y == 3).all())
        # 3: from an autograd hook
        p = torch.nn.Parameter(torch.zeros(n, device="cuda"))
        flat = torch.zeros(n, device="cuda"); p.grad = flat.view(-1)
        def hook(q):
            e = torch.cuda.Event(); e.record(); comm.wait_event(e)
            with torch.cuda.stream(comm):
                dist.all_reduce(flat)
        p.register_post_accumulate_grad_hook(hook)
        (p * (rank + 1)).sum().backward()
        torch.cuda.current_stream().wait_stream(comm); torch.cuda.synchronize()
        ok3 = bool((flat == 3).all())
        print(rank, n, ok1, ok2, ok3, float(flat[0]), flush=True)
    dist.destroy_process_group()
if __name__ == "__main__":
    mp.start_processes(worker, args=(2, port()), nprocs=2, join=True, start_method="spawn")
