# Round-2 evidence run (one gpurun call, ~5.5 min on one B200): bash tools/evidence_r02.sh, then python tools/update_profiles.py here.
# Every ncu capture is taken only after the same command has exited 0 without ncu.
set -x
K='regex:spmx_dev|spmm_|carry_|chain_|validate_|merge_|chunk_|exclusive_|count_|boundaries|ranges_|work_items|long_rows|l2_rows_probe'
python bench.py > gpurun_out/r02_bench_selfrun.json 2> gpurun_out/r02_bench_selfrun.err || exit 1
tail -c 600 gpurun_out/r02_bench_selfrun.json
python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bench_short.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" -c 700 --csv --log-file gpurun_out/r02_launches_bench_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/r02_ncu_bench.log 2>&1
for cfg in "c2 merge" "c3 nnz" "c4 merge" "c5 nnz"; do
  set -- $cfg
  python tools/prof_one.py $1 $2 fast 3 > gpurun_out/r02_prof_$1.log 2>&1 || exit 1
  ncu --set full --clock-control none --import-source on -k regex:spmm_chunk --launch-skip 2 -c 1 -o gpurun_out/r02_full_$1 -f python tools/prof_one.py $1 $2 fast 3 >> gpurun_out/r02_prof_$1.log 2>&1
done
python tools/prof_one.py c2 merge exact 3 > gpurun_out/r02_prof_c2_exact.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:long_row --launch-skip 2 -c 1 -o gpurun_out/r02_full_c2_longrow -f python tools/prof_one.py c2 merge exact 3 >> gpurun_out/r02_prof_c2_exact.log 2>&1
python tools/exp_hot_window.py c5 > gpurun_out/r02_exp_hot_window_c5.txt 2>&1 || exit 1
python tools/exp_hot_window.py c2 --iters 20 > gpurun_out/r02_exp_hot_window_c2.txt 2>&1
python tools/exp_hot_window.py c5 --profile > gpurun_out/r02_prof_c5_window.log 2>&1 || exit 1
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none -k regex:spmm_chunk -c 6 --csv --log-file gpurun_out/r02_c5_window_dram.csv python tools/exp_hot_window.py c5 --profile >> gpurun_out/r02_prof_c5_window.log 2>&1
SPMX_BENCH_SHARE_GPU=1 python bench.py --gpus 8 --steps 10 --allgather > gpurun_out/r02_share_c5_g8.json 2> gpurun_out/r02_share_c5_g8.err
for d in 8 16 32 64 128 256; do python tools/dev_bench.py c2 --d $d --modes fast,exact --strategies merge --iters 10 2>&1 | grep "==\|merge"; done > gpurun_out/r02_widths_c2.txt
python tools/dev_bench.py c1 c2 c3 c4 c5 --modes fast,exact --strategies row,nnz,merge,row-dyn --iters 10 > gpurun_out/r02_devbench_all.txt 2>&1
nvidia-smi --query-gpu=name,driver_version,clocks.max.sm,power.limit --format=csv > gpurun_out/r02_gpu.txt
ls -la gpurun_out/r02_* | head -40
