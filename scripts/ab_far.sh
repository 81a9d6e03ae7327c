# A/B of library builds (scratch_libs/*.so) on the far-field time: bash scripts/ab_far.sh cfg1 cfg4 -- base minb4 ...
mkdir -p gpurun_out
cfgs=(); libs=(); sep=0
for a in "$@"; do if [ "$a" = "--" ]; then sep=1; elif [ $sep = 0 ]; then cfgs+=("$a"); else libs+=("$a"); fi; done
for c in "${cfgs[@]}"; do for l in "${libs[@]}"; do
  ST_LIB_PATH=$PWD/scratch_libs/$l.so timeout 600 python bench.py --config $c --no-cpu-baseline --steps 4 --warmup 3 > gpurun_out/ab_${c}_$l.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/ab_${c}_$l.log').read().strip().splitlines()[-1]); s=d['step_phases_ms']['steps']; print('$c', '$l', 'step', round(d['ms_per_step'],2), 'far', [x[2] for x in s], 'near', s[-1][3])"
done; done
