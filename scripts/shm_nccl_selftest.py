"""Self-test of tests/cpp/shm_nccl.cpp: N processes on one GPU, all-reduce sum / max, broadcast, send / recv."""
import ctypes as C, os, sys, time
import numpy as np
import torch
lib = C.CDLL(os.environ["HLM_B200_NCCL_LIB"])
rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
idfile = "/tmp/shm_nccl_selftest.id"
uid = (C.c_uint8 * 128)()
if rank == 0:
    lib.ncclGetUniqueId(uid)
    open(idfile + ".tmp", "wb").write(bytes(uid)); os.rename(idfile + ".tmp", idfile)
else:
    while not os.path.exists(idfile): time.sleep(0.01)
    time.sleep(0.05)
    uid = (C.c_uint8 * 128).from_buffer_copy(open(idfile, "rb").read())
class Uid(C.Structure):
    _fields_ = [("b", C.c_uint8 * 128)]
u = Uid(); C.memmove(C.byref(u), uid, 128)
comm = C.c_void_p()
lib.ncclCommInitRank.argtypes = [C.POINTER(C.c_void_p), C.c_int, Uid, C.c_int]
assert lib.ncclCommInitRank(C.byref(comm), world, u, rank) == 0
lib.ncclAllReduce.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
x = torch.tensor([rank + 1, 10 * (rank + 1), 7, 0], dtype=torch.int32, device="cuda")
for it in range(3):
    y = x.clone()
    assert lib.ncclAllReduce(y.data_ptr(), y.data_ptr(), 4, 3, 0, comm, None) == 0
    print(rank, "sum", y.tolist(), flush=True)
k = torch.tensor([rank * 5 + 1, 100 - rank], dtype=torch.int64, device="cuda")
out = torch.zeros_like(k)
assert lib.ncclAllReduce(k.data_ptr(), out.data_ptr(), 2, 5, 2, comm, None) == 0
print(rank, "max", out.tolist(), flush=True)
lib.ncclCommDestroy.argtypes = [C.c_void_p]
lib.ncclCommDestroy(comm)
if rank == 0: os.remove(idfile)
