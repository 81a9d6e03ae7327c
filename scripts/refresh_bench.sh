# Refresh the committed bench lines (profiles/bench_<tag>_cfg*.json) and the launch list of
# the default bench command; plus the N=2 path smoke-tested on one GPU (gloo).
tag=${1:-r01}
mkdir -p gpurun_out
for c in cfg1 cfg0 cfg2 cfg4 cfg3; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_${tag}_$c.log 2>&1
  tail -1 gpurun_out/bench_${tag}_$c.log > gpurun_out/bench_${tag}_$c.json
done
timeout 600 python bench.py --impl reference > gpurun_out/bench_${tag}_reference.json 2>gpurun_out/bench_${tag}_reference.err
ST_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 > gpurun_out/bench_${tag}_n2_gloo.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_${tag}_bench_cfg1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
for f in gpurun_out/bench_${tag}_*.json; do echo "$f: $(head -c 300 $f)"; done
tail -2 gpurun_out/bench_${tag}_n2_gloo.log
# full ncu captures of the two evaluation kernels at cfg1 (current build)
ncu --set full --clock-control none --import-source on -k regex:k_neval -c 1 -o gpurun_out/neval_${tag} python scripts/profile_step.py cfg1 1 > gpurun_out/ncu_neval.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_far_list -c 1 -o gpurun_out/farlist_${tag} python scripts/profile_step.py cfg1 1 > gpurun_out/ncu_farlist.log 2>&1
