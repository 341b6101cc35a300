# bench.py under torchrun with 2 ranks sharing the one GPU of a gpurun box
# (gloo): checks the N > 1 plumbing (barriers, max over ranks, sharding, one
# JSON line from rank 0) that the driver's scaling run uses with NCCL.
mkdir -p gpurun_out/mr
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
TR="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533"
timeout 600 $TR bench.py --gpus 2 --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/mr/hero.json 2> gpurun_out/mr/hero.err; echo "hero rc=$?"
timeout 600 $TR bench.py --gpus 2 --steps 20 --warmup 3 --workload envs --envs 256 --no-cpu-baseline > gpurun_out/mr/envs.json 2> gpurun_out/mr/envs.err; echo "envs rc=$?"
timeout 600 $TR bench.py --gpus 2 --steps 10 --warmup 3 --workload slab --slab-particles 400000 --no-cpu-baseline > gpurun_out/mr/slab.json 2> gpurun_out/mr/slab.err; echo "slab rc=$?"
timeout 600 $TR bench.py --gpus 2 --steps 3 --warmup 3 --impl reference > gpurun_out/mr/ref.json 2> gpurun_out/mr/ref.err; echo "ref rc=$?"
for f in gpurun_out/mr/*.json; do echo "== $f"; wc -l < $f; tail -c 400 $f; echo; done
