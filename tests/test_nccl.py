"""NCCL binding of the native library (bcad_cu_nccl_unique_id /
bcad_cu_comm_init / bcad_cu_allreduce_adjoints) on the one GPU of a test box:
a 1-rank communicator must leave the adjoints unchanged, grouped buffers of
both dtypes included. The multi-rank sharding logic is covered on CPU by
tests/test_partition.py (gloo)."""
import pytest

pytestmark = pytest.mark.gpu


def test_single_rank_allreduce_is_identity():
    import torch
    from paper_1810_08297_b200 import native
    uid = native.nccl_unique_id()
    assert len(uid) == 128
    comm = native.Comm(1, uid, 0)
    try:
        a = torch.randn(3, 4096, device="cuda")
        b = torch.randn(17, device="cuda")
        a0, b0 = a.clone(), b.clone()
        comm.allreduce([a[0:1], a[1:2], a[2:3]])
        comm.allreduce([b])
        d = torch.randn(5, device="cuda", dtype=torch.float64)
        d0 = d.clone()
        comm.allreduce([d])
        torch.cuda.synchronize()
        assert torch.equal(a, a0) and torch.equal(b, b0) and torch.equal(d, d0)
    finally:
        comm.close()
