for i in 1 2 3; do python tools/profile_sweep.py --warm 3 --reps 3 > gpurun_out/ps_$i.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/ps_$i.json')); print(round(d['ms_sweep'],3), ' '.join('%s=%.2f'%(k['name'].split(':')[-1][:12],k['ms']) for k in d['kernels'][3:]))"; done
