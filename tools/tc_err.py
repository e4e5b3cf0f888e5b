#!/usr/bin/env python3
"""Max relative error (normwise protocol of tests/_parity.py) of the FP32 kernel
the library picks vs the oracle, for a few n / R / input distributions — used to
check the error-compensated TF32 kernel (JM_F32TC) against the 1e-5 FP32 bound."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import jm_synth  # noqa: E402
import oracle  # noqa: E402
import paper_1904_08555_b200 as jm  # noqa: E402
from tests._parity import max_rel_err  # noqa: E402

jm.jit_mat_init(0)
jm.jit_mat_set_stream(torch.cuda.current_stream().cuda_stream)
for n in [int(v) for v in sys.argv[1].split(",")]:
    for dist in ("hard", "shard", "bench"):
        x = jm_synth.generate(n, "f32", dist, 77 + n, 0, 203)
        errs = []
        for r in (1, 2, 3, 7, 100):
            want = oracle.run(x, r)
            got = jm.run(torch.from_numpy(x).cuda(), r, addend="ones", sync=True, variant="resident").cpu().numpy()
            errs.append(f"R={r}: {max_rel_err(got, want):.2e}")
        print(f"n={n} {dist}: " + ", ".join(errs), flush=True)
