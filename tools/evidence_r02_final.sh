# Round-2 closing run (one gpurun call): the GPU suite, smoke, the contract bench in its launch forms.
# bash tools/evidence_r02_final.sh   (the kernel source is unchanged since tools/evidence_r02.sh: ncu captures stand)
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/r02f_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/r02f_gputests.log
tail -4 gpurun_out/r02f_gputests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f_smoke.log 2>&1; tail -1 gpurun_out/r02f_smoke.log
python bench.py --impl reference > gpurun_out/r02f_bench_reference.json 2> gpurun_out/r02f_bench_reference.err
python bench.py > gpurun_out/r02f_bench_selfrun.json 2> gpurun_out/r02f_bench_selfrun.err
tail -c 400 gpurun_out/r02f_bench_selfrun.json
SPMX_BENCH_SHARE_GPU=1 python bench.py --gpus 2 --steps 5 > gpurun_out/r02f_share_c5_g2.json 2> gpurun_out/r02f_share_c5_g2.err
SPMX_BENCH_MG=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 5 --warmup 3 > gpurun_out/r02f_torchrun1_c5.json 2> gpurun_out/r02f_torchrun1_c5.err
python tools/cusparse_compare.py c2 c4 c3 c5 2>&1 | grep -v Warning | grep -v "A = torch" > gpurun_out/r02f_cusparse_compare.txt
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/r02f_gpu.txt
ls -la gpurun_out/r02f_*
