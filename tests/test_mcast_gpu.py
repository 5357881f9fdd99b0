"""The weight gradient fused with its all-reduce through an NVLink multicast object (include/smconv_mcast.h,
SURVEY.md §8(f) row 1), on ONE GPU: a multicast object bound to this GPU only (CUDA driver API through
cuda-python), so `multimem.red.add` adds into the single copy -- the kernel-side path of
the 8-GPU all-reduce (epilogue red for single-split TMA plans, reduce-kernel red otherwise) runs for real
and is compared with the oracle's full-batch dW (reading L10: SUM).  Integer inputs are bit-exact (the
cross-rank order of the in-switch adds cannot change exact integer sums); calling twice accumulates."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

SHAPES = [
    (128, 2, 2, 512, 512, 3, 3, 1, 1, 1, 1),   # VGG conv11: TMA (pairs in 3xTF32), epilogue red when one split
    (64, 16, 16, 64, 64, 3, 3, 1, 1, 1, 1),    # DWS split-K -> reduce-kernel red
    (32, 8, 8, 128, 256, 3, 3, 1, 1, 1, 1),    # TMA split-K
    (8, 8, 8, 4, 64, 3, 3, 1, 1, 1, 1),        # stem (GENERIC)
    (32, 6, 6, 48, 112, 5, 5, 1, 1, 2, 2),     # ragged channels (padded dW columns)
]


class DriverMulticast:
    """A 1-GPU NVLink multicast object made with the CUDA driver API (cuda-python): physical memory bound
    to the object, mapped at a unicast VA (read / zeroed by the test) and at the multicast VA the kernels
    add into.  Test infrastructure for the world-size-1 run; the product path uses torch symmetric memory
    (paper_2305_08819_b200/dp.py)."""

    def __init__(self, nbytes):
        from cuda.bindings import driver as cu
        self.cu = cu

        def ok(r, what=""):
            err = r[0] if isinstance(r, tuple) else r
            if err != cu.CUresult.CUDA_SUCCESS:
                raise RuntimeError("%s: %s" % (what, err))
            return r[1] if isinstance(r, tuple) and len(r) == 2 else r[1:] if isinstance(r, tuple) else None
        self.ok = ok
        dev = ok(cu.cuCtxGetDevice())
        sup = ok(cu.cuDeviceGetAttribute(cu.CUdevice_attribute.CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev))
        if not sup:
            raise RuntimeError("CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED = 0")
        mp = cu.CUmulticastObjectProp()
        mp.numDevices = 1
        mp.handleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        mp.flags = 0
        mp.size = nbytes
        gran = ok(cu.cuMulticastGetGranularity(mp, cu.CUmulticastGranularity_flags.CU_MULTICAST_GRANULARITY_RECOMMENDED),
                  "cuMulticastGetGranularity")
        size = (nbytes + gran - 1) // gran * gran
        mp.size = size
        self.size = size
        self.mc = ok(cu.cuMulticastCreate(mp), "cuMulticastCreate")
        ok(cu.cuMulticastAddDevice(self.mc, dev), "cuMulticastAddDevice")
        ap = cu.CUmemAllocationProp()
        ap.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
        ap.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
        ap.location.id = int(dev)
        ap.requestedHandleTypes = cu.CUmemAllocationHandleType.CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR
        self.mem = ok(cu.cuMemCreate(size, ap, 0), "cuMemCreate")
        ok(cu.cuMulticastBindMem(self.mc, 0, self.mem, 0, size, 0), "cuMulticastBindMem")
        acc = cu.CUmemAccessDesc()
        acc.location = ap.location
        acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
        self.uva = ok(cu.cuMemAddressReserve(size, gran, 0, 0), "cuMemAddressReserve")
        ok(cu.cuMemMap(self.uva, size, 0, self.mem, 0), "cuMemMap(unicast)")
        ok(cu.cuMemSetAccess(self.uva, size, [acc], 1), "cuMemSetAccess(unicast)")
        self.mva = ok(cu.cuMemAddressReserve(size, gran, 0, 0), "cuMemAddressReserve(mc)")
        ok(cu.cuMemMap(self.mva, size, 0, self.mc, 0), "cuMemMap(multicast)")
        ok(cu.cuMemSetAccess(self.mva, size, [acc], 1), "cuMemSetAccess(multicast)")

    def zero(self):
        self.ok(self.cu.cuMemsetD32(self.uva, 0, self.size // 4))

    def read(self, n):
        out = np.empty(n, np.float32)
        self.ok(self.cu.cuMemcpyDtoH(out.ctypes.data, self.uva, n * 4))
        return out


@pytest.fixture(scope="module")
def env():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import oracle
    from paper_2305_08819_b200 import build
    build.build()
    oracle.build()
    from paper_2305_08819_b200 import smconv as sm
    torch.cuda.set_device(0)
    torch.zeros(1, device="cuda")  # the primary context is current for the driver calls
    try:
        mc = DriverMulticast(64 << 20)
    except Exception as exc:  # pragma: no cover - depends on the GPU / fabric
        pytest.skip("no NVLink multicast object on this GPU: %s" % exc)
    return torch, oracle, sm, mc


@pytest.mark.parametrize("math", ["3xtf32", "tf32"])
@pytest.mark.parametrize("s", SHAPES, ids=lambda s: "x".join(map(str, s)))
def test_dw_mcast_equals_oracle(env, s, math, parity_log):
    torch, oracle, sm, mcb = env
    from paper_2305_08819_b200 import synth
    N, IH, IW, IC, OC, FH, FW, sh, sw, ph, pw = s
    OH, OW = sm.out_hw(IH, IW, FH, FW, (sh, sw), (ph, pw))
    n = OC * FH * FW * IC
    assert n * 4 <= mcb.size
    nb = sm.mcast_workspace_bytes(s, math)
    ws = torch.empty(max(nb, 16), dtype=torch.uint8, device="cuda")
    st = torch.cuda.current_stream().cuda_stream
    plan = sm.mcast_plan_describe(s, math)
    for integer in (1, 0):
        g = synth.rng(50, 1, salt=integer)
        X = synth.activations(g, N, IH, IW, IC, integer=integer)
        dY = synth.activations(g, N, OH, OW, OC, integer=integer)
        x, dy = torch.from_numpy(X).cuda(), torch.from_numpy(dY).cuda()
        ref = oracle.conv2d_bwd_filter(X, dY, (FH, FW), (sh, sw), (ph, pw))
        torch.cuda.synchronize()
        mcb.zero()
        sm.raw_call_mcast(x.data_ptr(), dy.data_ptr(), int(mcb.mva), s, math, ws.data_ptr(), nb, st)
        torch.cuda.synchronize()
        got = mcb.read(n).reshape(OC, FH, FW, IC)
        if integer:
            assert np.array_equal(got.astype(np.float64), ref), plan
            sm.raw_call_mcast(x.data_ptr(), dy.data_ptr(), int(mcb.mva), s, math, ws.data_ptr(), nb, st)  # accumulates
            torch.cuda.synchronize()
            assert np.array_equal(mcb.read(n).reshape(OC, FH, FW, IC).astype(np.float64), 2 * ref), plan
        else:
            e = float(np.max(np.abs(got - ref)) / np.max(np.abs(ref)))
            parity_log.append({"config": "mcast-world1", "layer": "x".join(map(str, s)), "op": "dw", "math": math,
                               "check": "random", "normwise": e, "tol": {"3xtf32": 1e-5, "tf32": 5e-3}[math],
                               "coverage": "whole tensor", "plan": plan})
            assert e <= {"3xtf32": 1e-5, "tf32": 5e-3}[math], (e, plan)
