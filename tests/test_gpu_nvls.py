"""the grad_W all-reduce fused into the GEMM epilogue through an
NVLS multicast address (multimem.red.add).  On one GPU the multicast object has a
single member, so the reduction adds the tile onto the zeroed buffer: grad_W must
equal the ordinary backward's exactly (0 + v = v; the test data has no subnormal
grad_W entries).  Skips where the device / driver offers no multicast object."""
import os

import numpy as np
import pytest
import torch

import synth
from gpu_helpers import to_bf16_cuda
from oracle.lsq_grad import cold_start_step

pytestmark = pytest.mark.gpu


class _DriverMulticast:
    """A one-device NVLS multicast object over a fresh physical allocation, built
    with the CUDA driver API (cuda-python): the unicast mapping is the grad_W
    buffer, the multicast mapping the address the epilogue reduces into.  Test
    plumbing only (multi-rank runs use torch symmetric memory, dist.SymmetricGradW)."""

    def __init__(self, nbytes, dev=0):
        import cuda.bindings.driver as d
        self.d = d

        def ok(r):
            err = r[0] if isinstance(r, tuple) else r
            if err != d.CUresult.CUDA_SUCCESS:
                raise RuntimeError(str(err))
            return r[1] if isinstance(r, tuple) and len(r) > 1 else None

        ok(d.cuInit(0))
        cudev = ok(d.cuDeviceGet(dev))
        if not ok(d.cuDeviceGetAttribute(d.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, cudev)):
            raise RuntimeError("device reports no multicast support")
        mp = d.CUmulticastObjectProp()
        mp.numDevices = 1
        mp.handleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        gran = ok(d.cuMulticastGetGranularity(mp, d.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED))
        size = (nbytes + gran - 1) // gran * gran
        mp.size = size
        self.mc_handle = ok(d.cuMulticastCreate(mp))
        ok(d.cuMulticastAddDevice(self.mc_handle, cudev))
        ap = d.CUmemAllocationProp()
        ap.type = d.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = dev
        ap.requestedHandleTypes = d.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        self.phys = ok(d.cuMemCreate(size, ap, 0))
        ok(d.cuMulticastBindMem(self.mc_handle, 0, self.phys, 0, size, 0))
        acc = d.CUmemAccessDesc()
        acc.location.type = d.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        acc.location.id = dev
        acc.flags = d.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uc = ok(d.cuMemAddressReserve(size, gran, 0, 0))
        ok(d.cuMemMap(self.uc, size, 0, self.phys, 0))
        ok(d.cuMemSetAccess(self.uc, size, [acc], 1))
        self.mc = ok(d.cuMemAddressReserve(size, gran, 0, 0))
        ok(d.cuMemMap(self.mc, size, 0, self.mc_handle, 0))
        ok(d.cuMemSetAccess(self.mc, size, [acc], 1))
        self.size = size

    def tensor(self, shape):
        """The unicast mapping as a float32 torch tensor (no copy)."""
        import numpy as np

        class _CAI:
            def __init__(s, ptr, shape):
                s.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<f4", "data": (ptr, False),
                                              "version": 3, "strides": None}
        return torch.as_tensor(_CAI(int(self.uc), shape), device="cuda")


def test_grad_w_multicast_reduction_one_device_driver_api():
    """The multimem.red epilogue itself, on a one-device multicast object: grad_W
    reduced through the multicast mapping lands in the unicast buffer and equals
    the ordinary backward's grad_W bit for bit."""
    import paper_2306_11987_b200 as i4
    N, D, C, k = 1024, 256, 512, 5
    try:
        mcb = _DriverMulticast(C * D * 4)
    except Exception as e:
        pytest.skip(f"no one-device multicast object: {e}")
    x, w = synth.activations(N, D, seed=5), synth.weights(C, D, seed=5)
    g = synth.grad_output(N, C, seed=5, dense=True)
    s_x, s_w = cold_start_step(x), cold_start_step(w)
    layer = i4.Int4Linear(N, D, C, k)
    Y = torch.empty(N, C, dtype=torch.float32, device="cuda")
    layer.forward(to_bf16_cuda(x), to_bf16_cuda(w), s_x, s_w, Y)
    dX = torch.empty(N, D, dtype=torch.float32, device="cuda")
    dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
    G = to_bf16_cuda(g)
    layer.backward(G, dX, dW, synth.PHILOX_SEED, call_id=4)
    torch.cuda.synchronize()
    buf = mcb.tensor((C, D))
    buf.zero_()
    dW2 = torch.full((C, D), 7.0, dtype=torch.float32, device="cuda")
    layer.backward(G, dX, dW2, synth.PHILOX_SEED, call_id=4, dw_multicast=int(mcb.mc))
    torch.cuda.synchronize()
    assert torch.equal(buf, dW)
    assert torch.all(dW2 == 7.0)                # dW untouched in this mode


def test_grad_w_multicast_reduction_single_rank():
    import torch.distributed as dist

    import paper_2306_11987_b200 as i4
    from paper_2306_11987_b200 import dist as pdist
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29517")
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    N, D, C, k = 1024, 256, 512, 5
    x, w = synth.activations(N, D, seed=3), synth.weights(C, D, seed=3)
    g = synth.grad_output(N, C, seed=3, dense=True)
    s_x, s_w = cold_start_step(x), cold_start_step(w)
    try:
        sym = pdist.SymmetricGradW(C * D, torch.device("cuda", 0))
    except Exception as e:                      # no symmetric-memory backend here
        pytest.skip(f"symmetric memory unavailable: {e}")
    if not sym.available:
        pytest.skip("no multicast object for this group (NVLS unsupported here)")
    layer = i4.Int4Linear(N, D, C, k)
    Y = torch.empty(N, C, dtype=torch.float32, device="cuda")
    layer.forward(to_bf16_cuda(x), to_bf16_cuda(w), s_x, s_w, Y)
    dX = torch.empty(N, D, dtype=torch.float32, device="cuda")
    dW = torch.empty(C, D, dtype=torch.float32, device="cuda")
    G = to_bf16_cuda(g)
    layer.backward(G, dX, dW, synth.PHILOX_SEED, call_id=4)
    torch.cuda.synchronize()
    ref = dW.clone()
    sym.zero_()
    dW2 = torch.full((C, D), 123.0, dtype=torch.float32, device="cuda")
    layer.backward(G, dX, dW2, synth.PHILOX_SEED, call_id=4, dw_multicast=sym.multicast(0))
    sym.barrier()
    torch.cuda.synchronize()
    got = sym.tensor.view(C, D)
    assert torch.equal(got, ref)
    assert torch.all(dW2 == 123.0)              # dW untouched in this mode
