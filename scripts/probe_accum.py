"""Probe: accuracy of tcgen05 fp32 accumulation for the LM-head logits (K = 4096) vs fp64 and vs an
emulated round-to-nearest per K=16 step.  Informs DESIGN.md's tolerance reading."""
import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kd_inputs as KI, paper_2603_01875_b200 as kd
V, d = 151936, 4096
W_t, W_s = KI.make_heads(V, d, 2048, seed=1000)
H_t, H_s = KI.make_hidden(256, W_t, W_s, seed=1001, head_seed=1000)
Wt = torch.from_numpy(W_t.view(np.int16)).cuda().view(torch.bfloat16)
Ht = torch.from_numpy(H_t.view(np.int16)).cuda().view(torch.bfloat16)
Z = kd.gemm_bf16_f32(Ht, Wt, M=256, N=V, K=d).double().cpu().numpy()
Wf = KI.bf16_to_f64(W_t); Hf = KI.bf16_to_f64(H_t)
Zx = Hf @ Wf.T
err = Z - Zx
top = Zx.argmax(axis=1)
print("tcgen05 fp32-acc |err| max %.3e  rms %.3e  mean(signed) %.3e" % (np.abs(err).max(), np.sqrt((err**2).mean()), err.mean()))
print("top-logit |err| max %.3e  median %.3e  (|z_top| median %.1f)" % (np.abs(err[np.arange(256), top]).max(), np.median(np.abs(err[np.arange(256), top])), np.median(Zx[np.arange(256), top])))
# RN emulation on 8 rows x all V
def acc16(W, h):
    acc = np.zeros(W.shape[0], np.float32)
    for k in range(0, W.shape[1], 16):
        acc = (acc.astype(np.float64) + W[:, k:k+16] @ h[k:k+16]).astype(np.float32)
    return acc.astype(np.float64)
e_rn = np.concatenate([acc16(Wf, Hf[i]) - Zx[i] for i in range(8)])
e_hw = err[:8].ravel()
print("rows 0-7: hw rms %.3e  RN16-emulated rms %.3e   hw==RN16 fraction %.4f" % (np.sqrt((e_hw**2).mean()), np.sqrt((e_rn**2).mean()), np.mean(np.isclose(e_hw, e_rn, rtol=0, atol=1e-12))))
# K order reversed (bias column enters last): same products, different accumulation order
Zr = kd.gemm_bf16_f32(Ht.flip(1).contiguous(), Wt.flip(1).contiguous(), M=256, N=V, K=d).double().cpu().numpy()
er = Zr - Zx
print("reversed K: |err| max %.3e rms %.3e ; top-logit max %.3e median %.3e" % (np.abs(er).max(), np.sqrt((er**2).mean()), np.abs(er[np.arange(256), top]).max(), np.median(np.abs(er[np.arange(256), top]))))
# bias-free part only (column 0 zeroed) to see the dependence on |acc|
H0 = Ht.clone(); H0[:, 0] = 0
Z0 = kd.gemm_bf16_f32(H0, Wt, M=256, N=V, K=d).double().cpu().numpy()
Z0x = Zx - np.outer(Hf[:, 0], Wf[:, 0])
e0 = Z0 - Z0x
print("no bias:    |err| max %.3e rms %.3e ; top-logit max %.3e" % (np.abs(e0).max(), np.sqrt((e0**2).mean()), np.abs(e0[np.arange(256), top]).max()))
# split K into 4 independent GEMMs summed in fp64 (promotion every 1024)
Zc = sum(kd.gemm_bf16_f32(Ht[:, c:c+1024].contiguous(), Wt[:, c:c+1024].contiguous(), M=256, N=V, K=1024).double().cpu().numpy() for c in range(0, d, 1024))
ec = Zc - Zx
print("4 chunks:   |err| max %.3e rms %.3e ; top-logit max %.3e" % (np.abs(ec).max(), np.sqrt((ec**2).mean()), np.abs(ec[np.arange(256), top]).max()))
