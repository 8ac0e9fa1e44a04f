python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python bench.py --no-cpu-baseline > gpurun_out/b2.json; python -c "
import json; d=json.loads(open('gpurun_out/b2.json').read().strip().splitlines()[-1]); print(d['ms_per_step'], d['e2e'], d['peak_hbm_mb'], d['gpu_launches'])"
for n in 1 2 8; do SDTW_E2E_CHUNKS=$n python bench.py --no-cpu-baseline --single-mode | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('chunks $n', d['e2e']['ms_per_step'])"; done
python bench.py --config c3 --no-cpu-baseline --single-mode | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c3', d['ms_per_step'], d['e2e']['ms_per_step'])"
