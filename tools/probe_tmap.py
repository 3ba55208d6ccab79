"""Probe cuTensorMapEncodeTiled constraints (box vs. global dims) on the GPU box."""
import torch
from cuda.bindings import driver as cu

torch.zeros(1, device="cuda")
buf = torch.empty(1 << 20, dtype=torch.float32, device="cuda")


def enc(dims, box, esz=4):
    strides = []
    acc = esz
    for d in dims[:-1]:
        acc *= d
        strides.append(acc)
    r = cu.cuTensorMapEncodeTiled(cu.CUtensorMapDataType.CU_TENSOR_MAP_DATA_TYPE_FLOAT32, len(dims), buf.data_ptr(),
                                  [cu.cuuint64_t(d) for d in dims], [cu.cuuint64_t(x) for x in strides],
                                  [cu.cuuint32_t(b) for b in box], [cu.cuuint32_t(1)] * len(dims),
                                  cu.CUtensorMapInterleave.CU_TENSOR_MAP_INTERLEAVE_NONE,
                                  cu.CUtensorMapSwizzle.CU_TENSOR_MAP_SWIZZLE_NONE,
                                  cu.CUtensorMapL2promotion.CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                                  cu.CUtensorMapFloatOOBfill.CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE)
    return r[0]


for dims, box in [([8, 7, 7, 2], [8, 9, 1, 1]), ([8, 7, 7, 2], [8, 7, 1, 1]), ([8, 9, 7, 2], [8, 9, 1, 1]),
                  ([8, 7, 7, 2], [16, 7, 1, 1]), ([96, 112, 112, 4], [96, 114, 1, 1])]:
    print(dims, box, enc(dims, box))
