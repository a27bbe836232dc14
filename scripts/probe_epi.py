"""Probe: per-tile epilogue timing of the fused passes (needs the KD_EPI_TIMING build: KD_LIB_PATH=.../libkdfused_tim.so).
Prints, per pass, the average cycles an epilogue warp spends per tile waiting for the MMA, in TMEM loads, and total
epilogue (loads + math + release)."""
import ctypes, os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import kd_inputs as KI, paper_2603_01875_b200 as kd
cfg = KI.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c4"]
n = 4096
W_t, W_s = KI.make_heads(cfg.vocab, cfg.d_t, cfg.d_s, seed=1000)
H_t, H_s = KI.make_hidden(n, W_t, W_s, seed=1001, head_seed=1000)
up = lambda b: torch.from_numpy(b.view(np.int16)).cuda().view(torch.bfloat16)
Ht, Hs, Wt, Ws = up(H_t), up(H_s), up(W_t), up(W_s)
L = kd.lib()
dbg = torch.zeros(2 * 148 * 16 * 4 + 2 * 148 * 4 + 2 * 148 * 4, dtype=torch.int64, device="cuda")
L.kd_debug_set_buffer.argtypes = [ctypes.c_void_p]
kd.fused_fwd_bwd(Ht, Wt, Hs, Ws, T=1.0, kind=cfg.kind)  # warm
torch.cuda.synchronize()
for name, pass_id in (("pass1+pass2", 0),):
    dbg.zero_()
    L.kd_debug_set_buffer(ctypes.c_void_p(dbg.data_ptr()))
    kd.profile_enable(True)
    kd.fused_fwd_bwd(Ht, Wt, Hs, Ws, T=1.0, kind=cfg.kind)
    torch.cuda.synchronize()
    prof = kd.profile_read()
    kd.profile_enable(False)
    L.kd_debug_set_buffer(None)
    allv = dbg.cpu().numpy().astype(np.float64)
    dd = allv[:2 * 148 * 16 * 4].reshape(2, 148, 16, 4)
    mm = allv[2 * 148 * 16 * 4:2 * 148 * 16 * 4 + 2 * 148 * 4].reshape(2, 148, 4)
    cta = dbg.cpu().numpy()[2 * 148 * 16 * 4 + 2 * 148 * 4:].reshape(2, 148, 4)
    for ps in range(2):
        c = cta[ps]
        c = c[c[:, 1] > 0]
        t0 = c[:, 0].min()
        st, en = (c[:, 0] - t0) / 1e3, (c[:, 1] - t0) / 1e3
        dur = en - st
        print(cfg.name, f"pass{ps + 1} CTAs {len(c)}: start spread {st.max():.1f} us, end min/median/max "
              f"{en.min():.1f}/{np.median(en):.1f}/{en.max():.1f} us, busy fraction {dur.sum() / (len(c) * en.max()):.3f}, "
              f"SM cycles/CTA median {np.median(c[:, 3]):.0f} (clock {np.median(c[:, 3] / (dur * 1e3)):.3f} GHz)")
        order = np.argsort(en)
        print("   earliest-finishing SMs", c[order[:6], 2].tolist(), "latest", c[order[-6:], 2].tolist())
    for ps in range(2):
        m = mm[ps]
        t = m[..., 3].sum()
        print(cfg.name, f"pass{ps + 1} MMA warp: tiles", int(t), "avg cycles/tile: wait-tempty %.0f, wait-full %.0f, issue span %.0f"
              % (m[..., 0].sum() / t, m[..., 1].sum() / t, m[..., 2].sum() / t))
    for ps in range(2):
        d = dd[ps]
        tiles = d[..., 3].sum()
        print(cfg.name, f"pass{ps + 1} epilogue warps: warp-tiles", int(tiles),
              "avg cycles/tile: wait-for-MMA %.0f, [coupled: TMEM loads | decoupled pass 2: teacher half] %.0f, [epilogue total | student half] %.0f"
              % (d[..., 0].sum() / tiles, d[..., 1].sum() / tiles, d[..., 2].sum() / tiles))
    print({k: round(v[1], 3) for k, v in prof.items()})
