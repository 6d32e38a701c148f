"""Debug driver: run single bf16 tensor-core forward cases, one per process,
and print status / parity against the oracle (tools only, not a test)."""
import subprocess
import sys

CASES = {
    "lstm256_b120_v20k": ("sst", 2, 256, 20000, 120),
    "lstm128_b120_v97": ("sst", 2, 128, 97, 120),
    "lstm256_b60_v97": ("sst", 2, 256, 97, 60),
    "lstm256_b400_v20k": ("sst", 2, 256, 20000, 400),
    "lstm128_b10": ("sst", 2, 128, 20000, 10),
    "lstm256_b1": ("sst", 2, 256, 20000, 1),
    "lstm256_b10": ("sst", 2, 256, 20000, 10),
    "lstm256_b120": ("sst", 2, 256, 97, 120),
    "dag128_b10": ("grid", 5, 128, 20000, 10),
    "dag256_b10": ("grid", 5, 256, 20000, 10),
    "fc256_b10": ("perfect7", 1, 256, 20000, 10),
    "fc512_b10": ("perfect7", 1, 512, 20000, 10),
}


def run(name):
    import os
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
    import numpy as np
    import oracle
    import synth
    import paper_2011_01383_b200 as cx
    from gpu_helpers import dev_f32, dev_i32, normwise_rel_err, weights_dev
    gen, cell, H, V, B = CASES[name]
    if gen == "sst":
        ch, _ = synth.sst_shaped_forest(B, 0)
        kind = synth.TREE
    elif gen == "grid":
        ch, _ = synth.grid_dags(B)
        kind = synth.DAG
    else:
        ch, _ = synth.perfect_forest(B, 7)
        kind = synth.TREE
    words = synth.word_ids(ch, V, 0, all_nodes=(cell == synth.DAGRNN))
    emb = synth.embedding(V, H, 0)
    ws_np, wd = weights_dev(cell, H, V)
    lin = cx.linearize(dev_i32(ch), kind)
    h, aux, _ = cx.forward(cell, H, wd, dev_f32(emb), dev_i32(words), lin, dtype=cx.BF16,
                           want_aux=True)
    st = cx.status(lin)
    print(name, "status", st, flush=True)
    os.makedirs("gpurun_out", exist_ok=True)
    np.save(f"gpurun_out/{name}_h.npy", h.cpu().numpy())
    np.save(f"gpurun_out/{name}_aux.npy", aux.cpu().numpy())
    import torch
    ws = next(b for k, b in cx._cx._ws._bufs.items() if k[1] == "fwd")
    n = ch.shape[1]
    hbw = ws[128:128 + 2 * n * H].view(torch.bfloat16).view(n, H).float().cpu().numpy()
    perm = lin.perm[:n].cpu().numpy()
    hb_ref = h.to(torch.bfloat16).float().cpu().numpy()[perm]
    badrows = np.nonzero(np.abs(hbw - hb_ref).max(axis=1) > 0)[0]
    print("hb rows differing from bf16(h_out):", len(badrows), badrows[:10].tolist(), flush=True)
    off = (128 + 2 * n * H + 255) // 256 * 256
    csw = ws[off:off + 4 * n * H].view(torch.float32).view(n, H).cpu().numpy()
    cs_ref = aux.cpu().numpy()[perm]
    badc = np.nonzero(np.abs(csw - cs_ref).max(axis=1) > 0)[0]
    print("cs rows differing from aux_out:", len(badc), badc[:10].tolist(), flush=True)
    for b in badrows[:3]:
        d = np.nonzero(hbw[b] != hb_ref[b])[0]
        print("   row", b, "units", d[:8].tolist(), "...", len(d), "hb", hbw[b][d[:4]].tolist(), "ref", hb_ref[b][d[:4]].tolist())
    if st[0] == 0:
        rst, _, rh, raux = oracle.forward(cell, H, V, ws_np, emb, words, ch, want_aux=True)
        hg = h.cpu().numpy()
        print(name, "err", normwise_rel_err(hg, rh), flush=True)
        ref = oracle.linearize(ch, kind)
        height = np.empty(len(hg), np.int64)
        height[ref["perm"]] = ref["height"]
        inv = np.empty(len(hg), np.int64)
        inv[ref["perm"]] = np.arange(len(hg))
        num = np.abs(hg - rh).max(axis=1) / np.maximum(np.abs(rh).max(axis=1), 1e-6)
        for lv in range(height.max() + 1):
            sel = height == lv
            bad = sel & (num > 2e-2)
            for b in np.nonzero(bad)[0][:2]:
                d = np.abs(hg[b] - rh[b]) > 2e-2 * np.abs(rh[b]).max()
                print("   input id", b, "bad units", np.nonzero(d)[0].tolist()[:40], "of", H)
                for k in range(ch.shape[0]):
                    c = ch[k][b]
                    if c >= 0 and aux is not None:
                        ea = np.abs(aux.cpu().numpy()[c] - raux[c]).max() / np.abs(raux[c]).max()
                        print("    child", c, "h err", num[c], "aux err", ea)
            print(f"  level {lv}: n={sel.sum()} maxerr={num[sel].max():.3e} bad={bad.sum()}",
                  "bad new ids:", inv[bad][:12].tolist(), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        run(sys.argv[1])
    else:
        for c in CASES:
            r = subprocess.run([sys.executable, __file__, c], capture_output=True, text=True, timeout=120)
            print((r.stdout + r.stderr[-400:]).strip(), flush=True)
