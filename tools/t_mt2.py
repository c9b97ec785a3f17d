import sys, os
sys.path.insert(0, os.getcwd())
import torch, paper_2509_01229_b200 as lqg
m, n, k = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
torch.manual_seed(0)
dw = lqg.DeviceWeights.quantize(torch.randn(n, k, device="cuda") * 0.02, 128)
q, ts = lqg.quantize_activations(torch.randn(m, k, device="cuda"))
acc = dw.gemm_accum(q)
torch.cuda.synchronize()
ref = (q.float() @ dw.dequant().float().T)
print(m, n, k, "max err", (acc.float() - ref).abs().max().item())
