import sys, numpy as np, torch
sys.path.insert(0, ".")
import jm_synth, oracle, paper_1904_08555_b200 as jm
from tests._parity import max_rel_err
jm.jit_mat_init(0); jm.jit_mat_set_stream(torch.cuda.current_stream().cuda_stream)
for n in (37, 38, 39, 41, 45, 49, 57):
    x = jm_synth.generate(n, "f32", "paper", 0, 0, 3)
    errs = []
    for r in (1, 2, 4, 6, 8, 16):
        want = oracle.run(x, r)
        got = jm.run(torch.from_numpy(x).cuda(), r, sync=True).cpu().numpy()
        nf = int((~np.isfinite(want)).sum())
        errs.append(f"R={r}: {max_rel_err(got, want):.1e} (nonfin {nf})")
    print(n, ", ".join(errs), flush=True)
