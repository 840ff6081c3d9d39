import sys, numpy as np, torch
sys.path.insert(0,'.'); sys.path.insert(0,'tests')
import oracle.ringflow_np as O
from paper_2605_28657_b200.latents import fill_normals, philox_key
for (seed, stream, step, tag, n) in [(123,456,9,"long",1_000_000), (77,0,0,"big",1_000_000), (77,1,0,"big",1_000_000)]:
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    st = torch.zeros(1, dtype=torch.int32, device="cuda")
    fill_normals([(philox_key(seed,stream,step,tag), out)], st)
    g = out.cpu().numpy(); r = O.normal(seed,stream,step,tag,(n,))
    bad = np.nonzero(g.view(np.uint64) != r.view(np.uint64))[0]
    print(tag, stream, "status", int(st.item()), "nbad", len(bad), "first", bad[:5])
    if len(bad):
        i = bad[0]; print("  got", g[i-2:i+3]); print("  ref", r[i-2:i+3])
        # is it a shift? compare g[i:] with r[i+k:]
        for k in range(-3,4):
            m = min(len(g)-i, len(r)-i-k) - 10
            if m > 0 and i+k >= 0: print("  shift",k, np.mean(g[i:i+m]==r[i+k:i+k+m]))
