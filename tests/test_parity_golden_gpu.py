"""The GPU step against fixtures the REFERENCE ITSELF produced (tests/golden/make_golden.py via oracle/_ref), at the
two sizes SURVEY 8(c) asks for beyond the small parity cases:

* ``w10b``: the benchmarked 10B width (paper_config depth 1: H3456, 24 heads x 144, text 64 x 4096), latent
  (4,8,8) -> 64 tokens, first-frame conditioning on;
* ``long480p``: long N at reduced width (H288 = 2 x 144, rope (48,48,48)) on the real 480p/2s coordinates,
  latent (7,60,104) -> 10,920 tokens -- the reference's Tape::l2norm_heads / mul_head_scalar / rope3d / mha and
  their backward (autodiff.cpp:719-899) at that length, inside the whole block.

fp32 mode: loss, velocity rows, every parameter gradient within 1e-4 normwise (max |gpu - ref| over the stored
entries / max |ref|, plus the relative error of the full-tensor norm).  bf16 mode: the same table is reported per
tensor (north_star: "bf16 error bounded and reported"), bounded at 5e-2, and written to $MGV_REPORT_DIR when set.
At 10B width the fp32 run is also compared with the numpy restatement on every entry."""
import json
import os

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden.make_golden import LONG_CASES, build_case
from tests.gpu_common import nerr, to_cfg, to_samples
from tests.test_oracle import check_against_golden

pytestmark = pytest.mark.gpu
GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
TOL = {"fp32": 1e-4, "bf16": 5e-2}


@pytest.fixture(scope="module")
def cases():
    return {}


def _case(cases, name):
    if name not in cases:
        cases[name] = build_case(name, LONG_CASES[name])
    return cases[name]


@pytest.mark.parametrize("name", sorted(LONG_CASES))
@pytest.mark.parametrize("prec", ["fp32", "bf16"])
def test_step_vs_reference_golden(cases, name, prec):
    from paper_2510_17519_b200.capi import Context
    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    cfg, P, text, samples = _case(cases, name)
    ctx = Context(0, prec)
    ctx.upload(to_cfg(cfg), P)
    out = ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True)
    ctx.close()
    errs = check_against_golden(out, g, samples)
    worst = max(errs, key=errs.get)
    print(f"{name}/{prec}: worst {worst} {errs[worst]:.3e}; loss {errs['loss']:.2e} V0 {errs['V0']:.2e}")
    rep = os.environ.get("MGV_REPORT_DIR")
    if rep:
        os.makedirs(rep, exist_ok=True)
        with open(os.path.join(rep, f"parity_{name}_{prec}.json"), "w") as f:
            json.dump({"case": name, "precision": prec, "N": int(samples[0].clean.shape[0]),
                       "metric": "max|gpu-ref| over stored entries / max|ref| (and full-norm rel. error)",
                       "worst": [worst, errs[worst]], "errors": errs}, f, indent=1, sort_keys=True)
    assert errs[worst] <= TOL[prec], (worst, errs[worst])


def test_w10b_fp32_every_entry(cases):
    """10B width, fp32 mode: every entry of V and of every gradient against the numpy restatement (pinned to the
    reference at this width by test_oracle.py)."""
    from paper_2510_17519_b200.capi import Context
    cfg, P, text, samples = _case(cases, "w10b")
    ref = O.flow_fwdbwd(P, cfg, samples, text, 8.0, grads=True)
    ctx = Context(0, "fp32")
    ctx.upload(to_cfg(cfg), P)
    out = ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True)
    ctx.close()
    errs = {"loss": abs(out["loss"] - ref["loss"]) / abs(ref["loss"]), "V0": nerr(out["V"][0], ref["V"][0])}
    for k, gv in ref["grads"].items():
        errs[k] = nerr(out["grads"][k], gv)
    worst = max(errs, key=errs.get)
    print(f"w10b fp32 every entry: worst {worst} {errs[worst]:.3e}")
    assert errs[worst] <= 1e-4, (worst, errs[worst])


@pytest.mark.parametrize("name,size,prec", [("w10b", 2, "fp32"), ("w10b", 4, "fp32"), ("w10b", 8, "fp32"),
                                            ("w10b", 8, "bf16"), ("long480p", 2, "fp32"), ("long480p", 2, "bf16")])
def test_tp_step_vs_reference_golden(cases, name, size, prec):
    """Megatron head/column TP against the reference's own fixtures at the benchmarked 10B width
    (24 heads over P = 2 / 4 / 8 ranks: 12 / 6 / 3 heads per rank, partitioned weights, the peer-memory exchange)
    and at 10,920 tokens: every rank of the group is emulated in one context on this GPU (mgv_ctx_set_tp(P, 0,
    NULL)); gradients come back in reference layout (all-gathered blocks, permutation undone)."""
    from paper_2510_17519_b200.capi import Context
    g = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    cfg, P, text, samples = _case(cases, name)
    ctx = Context(0, prec)
    ctx.set_tp(size)
    ctx.upload(to_cfg(cfg), P)
    out = ctx.flow_step(to_samples(samples), text, 8.0, grads=True, velocity=True)
    ctx.close()
    errs = check_against_golden(out, g, samples)
    worst = max(errs, key=errs.get)
    print(f"tp{size} {name}/{prec}: worst {worst} {errs[worst]:.3e}; loss {errs['loss']:.2e}")
    assert errs[worst] <= TOL[prec], (worst, errs[worst])
