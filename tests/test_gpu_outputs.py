"""GPU: output element types (fm_out_dtype) and their range check."""

import numpy as np
import pytest

from oracle import cnaive

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("odt", ["uint8", "int16", "uint16", "int32"])
def test_out_dtypes_bit_exact(odt):
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    rng = np.random.default_rng(31)
    imgs = rng.integers(0, 40, (3, 90, 77)).astype(np.uint8)
    se = rng.integers(0, 9, (9, 11))
    tdt = getattr(torch, odt)
    for mode in ("dilate", "erode"):
        if mode == "erode" and odt in ("uint8", "uint16"):
            continue   # erosion can go negative
        plan = MorphPlan(shape=(90, 77), se_values=se, se_lo=(-4, -5), mode=mode, img_dtype=torch.uint8,
                         img_min=0, img_max=39, fill=0 if mode == "dilate" else 39, batch=3, out_dtype=tdt)
        out, valid = plan.execute(torch.from_numpy(imgs).cuda())
        assert out.dtype == tdt
        host, hvalid = plan.execute_host(imgs)
        for i in range(3):
            ref, _ = cnaive.naive(imgs[i], None, se, None, (-4, -5), erode=(mode == "erode"),
                                  fill=0 if mode == "dilate" else 39)
            assert np.array_equal(out[i].cpu().numpy().astype(np.int64), ref)
            assert np.array_equal(host[i].numpy().astype(np.int64), ref)


def test_out_dtype_range_rejected():
    import torch
    from paper_2305_03018_b200.engine import MorphPlan
    with pytest.raises(ValueError):
        MorphPlan(shape=(32, 32), se_values=np.full((3, 3), 5), se_lo=(-1, -1), img_dtype=torch.uint8,
                  img_min=0, img_max=255, out_dtype=torch.uint8)
    with pytest.raises(ValueError):
        MorphPlan(shape=(32, 32), se_values=np.full((3, 3), 5), se_lo=(-1, -1), mode="erode",
                  img_dtype=torch.uint8, img_min=0, img_max=100, fill=100, out_dtype=torch.uint8)
