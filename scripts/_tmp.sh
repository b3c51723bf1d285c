python bench.py --no-cpu-baseline --no-graph > gpurun_out/bng.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bng.json').read().strip().splitlines()[-1]);print('c3 eager', round(d['value']), round(d['ms_per_step'],4), round(d['e2e']['value']))"
python - <<'PY'
import time, torch, numpy as np, sys
sys.path.insert(0,'.')
from bench import CONFIGS
from paper_1906_00091_b200 import DlrmConfig, init_model
from paper_1906_00091_b200.rng import RandomBatchSource
from paper_1906_00091_b200.trainer import StepEngine
c=CONFIGS['c3']; B=c['batch']
cfg=DlrmConfig(c['tables'],c['d'],c['bot'],c['top'],seed=0)
m=init_model(cfg,table_init='device')
src=RandomBatchSource(c['tables'],c['bot'][0],B,c['k'],c['fixed'],seed=1)
hb=src.next_batch()
eng=StepEngine(m,B,[B*c['k']]*8,lr=0.1)
eng.load(hb.dense,hb.offsets,hb.indices,hb.labels)
for _ in range(3): eng.launch()
torch.cuda.synchronize()
t0=time.perf_counter()
for _ in range(20): eng.launch()
t1=time.perf_counter()
torch.cuda.synchronize()
t2=time.perf_counter()
print('host issue per step us', (t1-t0)/20*1e6, 'total per step us', (t2-t0)/20*1e6)
PY
