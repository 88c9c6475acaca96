cat > gpurun_out/c1a.py <<'PY'
import torch
from paper_2504_09186_b200 import DenseTensor, contract_pair
from paper_2504_09186_b200.workloads import c1_cases
case=c1_cases()[0]; ia,ib,io=case.index_lists(); da,db=case.data()
a,b=DenseTensor(ia,da),DenseTensor(ib,db)
for _ in range(3): out=contract_pair(a,b,out_order=io)
torch.cuda.synchronize()
s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(20): out=contract_pair(a,b,out_order=io)
e.record(); e.synchronize(); print("ms/step", s.elapsed_time(e)/20)
PY
for mb in 2 3; do for ks in 16 8; do echo "minb=$mb ks=$ks"; TNC_STREAM_MINB=$mb TNC_STREAM_KS=$ks PYTHONPATH=. python gpurun_out/c1a.py; done; done
TNC_STREAM_MINB=3 TNC_STREAM_KS=8 python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -1
