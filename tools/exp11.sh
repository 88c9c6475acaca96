python -m pytest tests/test_gpu_stream.py -x -q 2>&1 | tail -3
python -m pytest tests/test_gpu_fullsize.py -x -q -k "c1" 2>&1 | tail -2
python bench.py --workload c1 --steps 10 --warmup 3 2>&1 | head -1 | cut -c1-300
python - <<'PY' > gpurun_out/c1a_plain.log 2>&1
import sys; sys.argv=['x']
import torch
from paper_2504_09186_b200 import DenseTensor, contract_pair
from paper_2504_09186_b200.workloads import c1_cases
case=c1_cases()[0]; ia,ib,io=case.index_lists(); da,db=case.data()
a,b=DenseTensor(ia,da),DenseTensor(ib,db)
for _ in range(3): contract_pair(a,b,out_order=io)
torch.cuda.synchronize(); print("ok")
PY
ncu --set full --clock-control none --import-source on -k regex:stream_kernel -c 1 -o gpurun_out/stream_c1a2 python - <<'PY' > gpurun_out/ncu_stream.log 2>&1
import torch
from paper_2504_09186_b200 import DenseTensor, contract_pair
from paper_2504_09186_b200.workloads import c1_cases
case=c1_cases()[0]; ia,ib,io=case.index_lists(); da,db=case.data()
a,b=DenseTensor(ia,da),DenseTensor(ib,db)
contract_pair(a,b,out_order=io); torch.cuda.synchronize()
PY
echo "ncu rc=$?"
