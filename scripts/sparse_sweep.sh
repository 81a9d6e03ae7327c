# far-event deferral threshold (ST_FAR_SPARSE) sweep: step / far / near ms per config
for c in cfg1 cfg4 cfg2; do for t in 16 20 24 28; do
  ST_FAR_SPARSE=$t timeout 600 python bench.py --config $c --no-cpu-baseline --steps 4 > gpurun_out/sp_${c}_$t.log 2>&1
  tail -1 gpurun_out/sp_${c}_$t.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); s=d['step_phases_ms']['steps']; print('$c', 'sparse_max', $t, 'step', round(d['ms_per_step'],2), 'far', round(sum(x[2] for x in s)/len(s),2), 'near', round(sum(x[3] for x in s)/len(s),2))"
done; done
