"""Probe: tcgen05 fp32 accumulation error over a long K (the dh GEMM sums over V = 151936) and the
effect of splitting K into independent accumulators summed outside (split-K 'promotion')."""
import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kd_inputs as KI, paper_2603_01875_b200 as kd
torch.manual_seed(0)
V, M, N = 151936, 256, 256
# G-like rows: peaked, zero-sum; B = W_s-like columns incl. a bias column with large values
p = torch.softmax(torch.randn(M, V, dtype=torch.float64) * 3, dim=1)
q = torch.softmax(torch.randn(M, V, dtype=torch.float64) * 3, dim=1)
G = (q - p)
Gh = G.float().to(torch.bfloat16); Gl = (G.float() - Gh.float()).to(torch.bfloat16)
W = (torch.randn(V, N, dtype=torch.float64) * 0.03); W[:, 0] = torch.from_numpy(-np.log(np.random.default_rng(0).permutation(V) + 1.0)); W[:, 0] -= W[:, 0].mean()
Wb = W.to(torch.bfloat16)
ref = (Gh.double() + Gl.double()) @ Wb.double()
def run(k_split):
    out = torch.zeros(M, N, dtype=torch.float64)
    for c in range(k_split):
        a, b = V * c // k_split, V * (c + 1) // k_split
        a -= a % 64; b = V if c == k_split - 1 else b - b % 64
        for plane in (Gh, Gl):
            out += kd.gemm_bf16_f32(plane[:, a:b].contiguous().cuda(), Wb[a:b].contiguous().cuda(), M=M, N=N, K=b - a, b_mn_major=True).double().cpu()
    return out
for ks in (1, 4, 16, 64):
    e = run(ks) - ref
    rel = e.abs() / (1e-5 + 2e-3 * ref.abs())
    print(f"k_split {ks:3d}: max|err| {e.abs().max():.3e} col0 max {e[:,0].abs().max():.3e} rms {e.pow(2).mean().sqrt():.3e} worst err/tol {rel.max():.2f}")
