"""C5 grouped expert GEMM timing (bench.py grouped_experts, standalone; development aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2603_08713_b200 as M
import bench
class A: pass
from paper_2603_08713_b200 import parallel as P
r = bench.grouped_experts(torch, M, P, torch.device("cuda", 0), A())
for k, v in r.items():
    print(k, v)
