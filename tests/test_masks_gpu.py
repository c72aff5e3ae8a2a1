"""General unit-aligned condition masks in the device training step (apply_condition_mask, flowtrain.cpp:61-100):
any set of whole latent units, with condition latents that differ from the clean rows, against the oracle (whose
mask handling test_oracle.py pins to the reference); and the reference's InputErrors."""
import numpy as np
import pytest

from oracle import oracle as O
from tests.gpu_common import nerr, to_cfg, to_samples
from tests.test_oracle import mask_case

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind", ["last", "two", "none"])
@pytest.mark.parametrize("prec,tol", [("fp32", 1e-4), ("bf16", 5e-2)])
def test_general_mask_step(kind, prec, tol):
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = mask_case(kind)
    ref = O.flow_fwdbwd(P, cfg, samples, text, 8.0, grads=True)
    ctx = Context(0, prec)
    ctx.upload(to_cfg(cfg), P)
    out = ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True)
    ctx.close()
    errs = {"loss": abs(out["loss"] - ref["loss"]) / abs(ref["loss"])}
    for i in range(len(samples)):
        errs[f"V{i}"] = nerr(out["V"][i], ref["V"][i])
    for k, g in ref["grads"].items():
        errs[k] = nerr(out["grads"][k], g)
    worst = max(errs, key=errs.get)
    print(f"mask {kind}/{prec}: worst {worst} {errs[worst]:.3e}")
    assert errs[worst] <= tol, (worst, errs[worst])


def test_mask_errors():
    from paper_2510_17519_b200.capi import Context, FlowSample, InputError
    cfg, P, text, samples = mask_case("last")
    ctx = Context(0, "fp32")
    ctx.upload(to_cfg(cfg), P)
    s = samples[1]
    bad = s.mask.copy()
    bad[np.argmax(s.coords[:, 0] == 2)] = 0  # a partly conditioned unit (flowtrain.cpp:66-76)
    with pytest.raises(InputError, match="whole latent units"):
        ctx.flow_step([FlowSample(s.dims, s.coords, s.clean, s.noise, s.t, bad)], text, 8.0)
    # conditioned tokens without condition latents (flowtrain.cpp:77-80): a sample built at the C level
    import ctypes
    from paper_2510_17519_b200.capi import mgv_flow_sample
    fs = FlowSample(s.dims, s.coords, s.clean, s.noise, s.t, s.mask)
    cs = (mgv_flow_sample * 1)(fs.to_c())
    cs[0].condition_latents = None
    tx = np.ascontiguousarray(text, dtype=np.float64)
    loss, gn = ctypes.c_double(), ctypes.c_double()
    with pytest.raises(InputError, match="lacks clean latents"):
        ctx._check(ctx._L.mgv_flow_step(ctx.h, 1, cs, tx.ctypes.data, tx.shape[0], 8.0, ctypes.byref(loss),
                                        ctypes.byref(gn), None, None))
    ctx.close()
