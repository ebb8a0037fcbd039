"""Replays the N>1 bench stages on 2 processes sharing cuda:0 with an error
check after every call (dev tool)."""
import os
import socket
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402


def worker(rank, world, port, n):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    import paper_2508_03760_b200 as fc
    from paper_2508_03760_b200.dist import QComm
    from bench import spiky_bf16
    dev = torch.device("cuda", 0)
    cfg = fc.QuantConfig(4, group_size=128, chunk_size=128, scheme=fc.Scheme.SPIKE_RESERVING)
    comm = QComm(max_elems=n, config=cfg, timeout_s=60.0, oneshot_max_elems=1 << 18)
    x = spiky_bf16(n, 1000 + rank, dev)
    y = torch.empty_like(x)
    ref = comm.all_reduce(x, check=True, algo="two_step").clone()

    def step(name, fn, k=1):
        for i in range(k):
            torch.cuda.synchronize()
            dist.barrier()
            fn()
            torch.cuda.synchronize()
            try:
                comm.check()
            except Exception as e:
                print(f"rank {rank}: {name} call {i}: {e}", flush=True)
                return False
        return True

    step("two_step", lambda: comm.all_reduce(x, out=y, algo="two_step"), 3)
    for i in range(6):
        ok = step("pipelined", lambda: comm.all_reduce(x, out=y, algo="pipelined"))
        same = bool(torch.equal(y, ref))
        print(f"rank {rank}: pipelined {i} ok={ok} equal_two_step={same}", flush=True)
    # probe: garbage into the peer's buffer, as the bench does
    probe = min(256 << 20, comm.buffer_bytes // 2 // 16 * 16)
    src = torch.empty(probe, dtype=torch.uint8, device=dev)
    peer = (rank + 1) % world
    lib = fc._lib.lib()
    step("probe", lambda: fc._lib.check(lib.fc2_copy_bytes(comm.buffer_ptr(peer), src.data_ptr(), probe, 0,
                                                            torch.cuda.current_stream().cuda_stream)), 3)
    step("two_step after probe", lambda: comm.all_reduce(x, out=y, algo="two_step"), 2)
    print(f"rank {rank}: after probe equal={bool(torch.equal(y, ref))}", flush=True)
    for i in range(3):
        ok = step("pipelined after probe", lambda: comm.all_reduce(x, out=y, algo="pipelined"))
        print(f"rank {rank}: pipelined-after-probe {i} ok={ok} equal={bool(torch.equal(y, ref))}", flush=True)
    ok = step("oneshot", lambda: comm.all_reduce(x[:32768], out=y[:32768]), 3)
    print(f"rank {rank}: done", flush=True)
    comm.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 25
    s = socket.socket(); s.bind(("127.0.0.1", 0)); port = s.getsockname()[1]; s.close()
    mp.start_processes(worker, args=(2, port, n), nprocs=2, start_method="spawn")
