"""Argument checks of the Python binding (paper_2503_08217_b200/s3r.py) that run
before any pointer crosses the C ABI: wrong dtype / shape / layout raise
ValueError (the kernels index buffers by the sizes in the structs)."""
import pytest
import torch

from paper_2503_08217_b200 import s3r


def test_req_accepts_matching_tensor():
    s3r._req(torch.zeros(5, 4), "x", torch.float32, (5, 4))
    s3r._req(None, "x", torch.float32, (5, 4), optional=True)


@pytest.mark.parametrize("t, why", [
    (torch.zeros(5, 4, dtype=torch.float64), "dtype"),
    (torch.zeros(5, 3), "shape"),
    (torch.zeros(4, 5).t(), "contiguous"),
    (None, "None"),
    ([0.0] * 20, "torch.Tensor"),
])
def test_req_rejects(t, why):
    with pytest.raises(ValueError, match=why):
        s3r._req(t, "x", torch.float32, (5, 4))


def test_req_rejects_cpu_tensor_for_device():
    with pytest.raises(ValueError, match="expected cuda:0"):
        s3r._req(torch.zeros(5, 4), "x", torch.float32, (5, 4), device=0)


def test_scene_check_shapes():
    n = 7
    ds = s3r.DeviceScene(torch.zeros(n, 4), torch.zeros(n, 4), torch.zeros(n, 4),
                         torch.zeros(n, 4), torch.zeros(n, dtype=torch.int32),
                         torch.zeros(n, 2), torch.zeros(n, 2), 1)
    ds.check()                                   # shapes and dtypes (device not checked)
    ds.instance_ids = torch.zeros(n, dtype=torch.int64)
    with pytest.raises(ValueError, match="instance_ids"):
        ds.check()
    ds.instance_ids = torch.zeros(n, dtype=torch.int32)
    ds.life = torch.zeros(n, 3)
    with pytest.raises(ValueError, match="life"):
        ds.check()


def test_table_check():
    with pytest.raises(ValueError, match="3x4"):
        s3r._req_table(torch.zeros(2, 12), "tables[0]", 3, 0)
