python -m pytest tests -m gpu -x -q > gpurun_out/t19.log 2>&1; tail -2 gpurun_out/t19.log
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench19.log 2>&1; tail -1 gpurun_out/bench19.log | cut -c1-300
TMB_NO_TTM2=1 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench19b.log 2>&1; tail -1 gpurun_out/bench19b.log | cut -c1-300
python -c "
import json
a=json.loads(open('gpurun_out/bench19.log').read().strip().splitlines()[-1]); b=json.loads(open('gpurun_out/bench19b.log').read().strip().splitlines()[-1])
print('fit', a['fit'], b['fit'], 'rel', a['rel_err'], b['rel_err'], 'identical', a['fit']==b['fit'] and a['rel_err']==b['rel_err'])"
