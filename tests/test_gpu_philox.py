"""The oracle's Philox4x32-10 (R18, R19) against curand's DEVICE implementation
on all four counter words and both key words.

The CPU pin (test_oracle_pins.py::test_philox_matches_curand_host_generator)
reaches counter words c0 and c2 only (the host generator's stream layout); the
transmission draws of the voxel march use all four (pulse lo/hi, subray, voxel
id).  Here a tiny kernel calls curand_Philox4x32_10(c, k) -- curand's own
device code, compiled with nvcc into a throw-away library -- on random counters
and keys, and every output word must equal the oracle's.
"""
import ctypes
import os
import subprocess
import tempfile

import numpy as np
import pytest

import oracle
from gpu_util import torch_cuda

pytestmark = pytest.mark.gpu

_SRC = r"""
#include <curand_kernel.h>
__global__ void k(const uint4* c, const uint2* key, uint4* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = curand_Philox4x32_10(c[i], key[i]);
}
extern "C" int run(const void* c, const void* key, void* out, int n) {
  k<<<(n + 127) / 128, 128>>>((const uint4*)c, (const uint2*)key, (uint4*)out, n);
  return (int)cudaDeviceSynchronize();
}
"""


def _curand_device_lib():
    d = tempfile.mkdtemp()
    src, so = os.path.join(d, "p.cu"), os.path.join(d, "p.so")
    with open(src, "w") as f:
        f.write(_SRC)
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a",
                           "-shared", "-Xcompiler", "-fPIC", src, "-o", so])
    return ctypes.CDLL(so)


def test_philox_all_counter_words_match_curand_device():
    torch = torch_cuda()
    lib = _curand_device_lib()
    rng = np.random.default_rng(11)
    n = 4096
    ctr = rng.integers(0, 2**32, (n, 4), dtype=np.uint64).astype(np.uint32)
    key = rng.integers(0, 2**32, (n, 2), dtype=np.uint64).astype(np.uint32)
    # the layouts the library uses: (pulse lo, pulse hi, subray, voxel id) and
    # key (seed lo, seed hi ^ stream tag), plus edge words
    ctr[:8] = [[0, 0, 0, 0], [0xFFFFFFFF] * 4, [1, 2, 3, 4], [5, 1, 18, 6399999],
               [123456789, 0, 90, 0], [0, 0xFFFFFFFF, 0, 0xFFFFFFFF], [7, 0, 0, 1], [0, 1, 0, 0]]
    key[:4] = [[0, 0], [0, 1], [0xFFFFFFFF, 0xFFFFFFFF], [7, 2]]
    c_d = torch.from_numpy(ctr.view(np.int32)).cuda()
    k_d = torch.from_numpy(key.view(np.int32)).cuda()
    o_d = torch.zeros((n, 4), dtype=torch.int32, device="cuda")
    assert lib.run(ctypes.c_void_p(c_d.data_ptr()), ctypes.c_void_p(k_d.data_ptr()),
                   ctypes.c_void_p(o_d.data_ptr()), n) == 0
    got = o_d.cpu().numpy().view(np.uint32)
    for i in range(n):
        ref = oracle.philox4x32_10(ctr[i], key[i])
        assert np.array_equal(got[i], ref), (i, ctr[i], key[i], got[i], ref)
