python bench.py --workload c1 --steps 10 --warmup 3 2>&1 | head -1
python - <<'PY'
import torch, time
from paper_2504_09186_b200 import DenseTensor, contract_pair
from paper_2504_09186_b200.workloads import c1_cases
case=c1_cases()[0]; ia,ib,io=case.index_lists(); da,db=case.data()
a,b=DenseTensor(ia,da),DenseTensor(ib,db)
for _ in range(3): out=contract_pair(a,b,out_order=io)
torch.cuda.synchronize()
for rep in range(3):
    s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10): out=contract_pair(a,b,out_order=io)
    e.record(); e.synchronize(); print("ms/step", s.elapsed_time(e)/10)
t0=time.perf_counter()
for _ in range(10): out=contract_pair(a,b,out_order=io)
torch.cuda.synchronize(); print("wall ms/step", (time.perf_counter()-t0)*100)
PY
