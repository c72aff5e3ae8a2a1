"""Deep-stack weights for the full-depth tools: dit::init_dit_params(paper_config(depth=1), Rng(1)) plus the gate
opening from Rng(2), generated once by mgv_params_init and downloaded, with that one block's arrays
shared by every block name of a depth-D stack.  Host memory stays ~1.6 GB (fp64, one block) while the device holds D
independent copies -- the per-block kernels, memory and timing do not depend on the weight values."""
import math


def shared_stack_params(depth: int, device: int = 0) -> dict:
    from paper_2510_17519_b200.capi import Context, paper_config
    cfg1 = paper_config(depth=1)
    gs = 0.2 * math.sqrt(12.0 / cfg1.hidden)
    c = Context(device, "fp32")
    c.init_params(cfg1, seed=1, gate_seed=2, gate_std=gs, gate_b_std=gs / 4)
    one = c.download()
    c.close()
    params = {k: v for k, v in one.items() if not k.startswith("dit.blk.")}
    for i in range(depth):
        for k, v in one.items():
            if k.startswith("dit.blk.0."):
                params[f"dit.blk.{i}." + k[len("dit.blk.0."):]] = v
    return params
