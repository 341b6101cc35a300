# bench.py under torchrun with 2 ranks sharing the one GPU of a gpurun box
# (gloo for the collectives): checks the N > 1 plumbing (barriers, max over
# ranks, sharding, one JSON line from rank 0) that the driver's scaling run
# uses with NCCL, and the single-bed slab path with both exchanges (host
# point-to-point and the peer-memory mailboxes, CUDA IPC within one device).
mkdir -p gpurun_out/mr
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $TR bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline --halo host > gpurun_out/mr/bed1m_host.json 2> gpurun_out/mr/bed1m_host.err; echo "bed1m host rc=$?"
timeout 600 $TR bench.py --gpus 2 --steps 20 --warmup 3 --no-cpu-baseline --halo p2p > gpurun_out/mr/bed1m_p2p.json 2> gpurun_out/mr/bed1m_p2p.err; echo "bed1m p2p rc=$?"
timeout 600 $TR bench.py --gpus 2 --steps 50 --warmup 5 --workload hero50k --no-cpu-baseline > gpurun_out/mr/hero.json 2> gpurun_out/mr/hero.err; echo "hero rc=$?"
timeout 600 $TR bench.py --gpus 2 --steps 20 --warmup 3 --workload envs --envs 256 --no-cpu-baseline > gpurun_out/mr/envs.json 2> gpurun_out/mr/envs.err; echo "envs rc=$?"
timeout 600 $TR bench.py --gpus 2 --steps 10 --warmup 3 --workload slab --slab-particles 400000 --no-cpu-baseline --halo p2p > gpurun_out/mr/slab_p2p.json 2> gpurun_out/mr/slab_p2p.err; echo "slab p2p rc=$?"
timeout 600 $TR bench.py --gpus 2 --steps 3 --warmup 3 --impl reference > gpurun_out/mr/ref.json 2> gpurun_out/mr/ref.err; echo "ref rc=$?"
for f in gpurun_out/mr/*.json; do echo "== $f"; python -c "
import json,sys
try:
    d=json.load(open('$f')); print({k: d.get(k) for k in ('n_gpus','value','ms_per_step','scaling')}, d.get('run',{}).get('halo'), d.get('run',{}).get('parallelism'))
except Exception as e: print('bad', e)"; tail -2 ${f%.json}.err; done
