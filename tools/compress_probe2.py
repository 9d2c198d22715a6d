"""Development probe (not product): B200 generic compressible memory (cuMemCreate with
CU_MEM_ALLOCATION_COMP_GENERIC) holding the pJDS C3 jagged col / val arrays: written by an SM copy,
read by an SM reduction; ncu dram__bytes_read.sum of the reductions shows whether the matrix
stream would come back from DRAM in fewer bytes.  Prints the granted compression type."""
import os, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from cuda.bindings import driver as cu
import inputs
import paper_1112_5588_b200 as pj

torch.cuda.init()
torch.empty(1, device="cuda")
dev = 0


def chk(r):
    if isinstance(r, tuple):
        err, *rest = r
    else:
        err, rest = r, []
    assert err == cu.CUresult.CUDA_SUCCESS, err
    return rest[0] if len(rest) == 1 else rest


class Arr:
    def __init__(self, ptr, n, typestr):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3, "strides": None}


def comp_alloc(nbytes):
    prop = cu.CUmemAllocationProp()
    prop.type = cu.CUmemAllocationType.CU_MEM_ALLOCATION_TYPE_PINNED
    prop.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    prop.location.id = dev
    prop.allocFlags.compressionType = cu.CUmemAllocationCompType.CU_MEM_ALLOCATION_COMP_GENERIC
    gran = chk(cu.cuMemGetAllocationGranularity(prop, cu.CUmemAllocationGranularity_flags.CU_MEM_ALLOC_GRANULARITY_RECOMMENDED))
    size = (nbytes + gran - 1) // gran * gran
    h = chk(cu.cuMemCreate(size, prop, 0))
    got = chk(cu.cuMemGetAllocationPropertiesFromHandle(h))
    ptr = chk(cu.cuMemAddressReserve(size, 0, 0, 0))
    chk(cu.cuMemMap(ptr, size, 0, h, 0))
    acc = cu.CUmemAccessDesc()
    acc.location.type = cu.CUmemLocationType.CU_MEM_LOCATION_TYPE_DEVICE
    acc.location.id = dev
    acc.flags = cu.CUmemAccess_flags.CU_MEM_ACCESS_FLAGS_PROT_READWRITE
    chk(cu.cuMemSetAccess(ptr, size, [acc], 1))
    return int(ptr), size, got.allocFlags.compressionType


n, rp, col, val = inputs.config_crs(os.environ.get("CFG", "C3"))
A = pj.PjdsMatrix.from_crs(n, rp, col, val, block_rows=128, symmetric=True)
e = A.export()
del A, rp, col, val
for name, arr in (("zeros", np.zeros(len(e["col"]), np.int32)), ("col", e["col"]), ("val", e["val"])):
    src = torch.from_numpy(arr).cuda()
    ptr, size, ctype = comp_alloc(src.numel() * src.element_size())
    ts = "<i4" if arr.dtype == np.int32 else "<f8"
    t = torch.as_tensor(Arr(ptr, src.numel(), ts), device="cuda")
    t.copy_(src)  # SM writes into compressible memory
    torch.cuda.synchronize()
    del src
    torch.cuda.empty_cache()
    print(f"{name} compressible={ctype} bytes={arr.nbytes}", flush=True)
    for _ in range(2):
        s = t.sum()
        torch.cuda.synchronize()
