"""Two slab ranks (gloo, one GPU) stepping with the peer-memory exchange and
halo, for compute-sanitizer --target-processes all (memcheck / racecheck):
the mailbox pack, signal, wait and append kernels and the per-sweep halo."""
import os
import sys

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
import torch.multiprocessing as mp


def worker(rank, world, port):
    import torch.distributed as td
    from test_slab import _bed
    from paper_2306_01369_b200.slab import SlabBed

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    td.init_process_group("gloo", rank=rank, world_size=world)
    bed = SlabBed(_bed(), rank=rank, world=world, device=0, backend="gloo", resort_every=2, halo="p2p")
    reps = bed.run(3)
    print("rank", rank, "ok", reps[-1].n_contacts, bed.ghosts, flush=True)
    bed.close()
    td.destroy_process_group()


if __name__ == "__main__":
    mp.spawn(worker, args=(2, 29611), nprocs=2, join=True)
