#!/usr/bin/env python3
"""Run a list of update configurations once each, for one `ncu` capture of all of them.

    ncu --set full --clock-control none --import-source on -k regex:k_update -o REP \\
        python tools/ncu_configs.py 16:f64:1048576:100:resident 32:f32:262144:1:streaming ...

Each argument is n:dtype:batch:repeat:variant (variant = resident | streaming |
auto | generic | latency).  Inputs are the `bench` distribution filled on the device;
every configuration is warmed (compiled) before the captured launch, so the
NVRTC compile never lands inside a capture.  Prints the key info per config
(regs, smem, tile) as JSON lines so a summary can be matched to its config.
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch

    import paper_1904_08555_b200 as jm
    torch.cuda.init()
    jm.jit_mat_init(0)
    flags = {"resident": jm.JM_FLAG_RESIDENT, "streaming": jm.JM_FLAG_STREAMING, "auto": 0, "generic": 0,
             "latency": jm.JM_FLAG_LATENCY}
    for spec in sys.argv[1:]:
        n, dt, b, r, v = spec.split(":")
        n, b, r = int(n), int(b), int(r)
        tdt = torch.float64 if dt == "f64" else torch.float32
        x = torch.empty(b, n, n, dtype=tdt, device="cuda")
        y = torch.empty_like(x)
        jm.jit_mat_fill(n, dt, 1, 0x0019040855, 0, b, x.data_ptr())
        kind = "generic" if v == "generic" else "specialized"
        var = jm.jit_mat_prepare_for(n, dt, r, flags=flags[v], kind=kind) if kind == "specialized" else None
        jm.jit_mat_run_ex(n, dt, b, r, x.data_ptr(), y.data_ptr(), kind=kind, flags=flags[v] | jm.JM_FLAG_SYNC)
        info = [k for k in jm.jit_mat_key_info() if k["op"] == 0 and k["n"] == n
                and k["dtype"] == (1 if dt == "f64" else 0) and k["kind"] == (1 if kind == "generic" else 0)
                and k["addend"] == 0 and (var is None or k["variant"] == var)]
        print(json.dumps({"spec": spec, "variant": var, "keys": info}), flush=True)
        del x, y
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
