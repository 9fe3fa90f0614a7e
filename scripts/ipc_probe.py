"""Probe: which cudaMalloc sizes can be exported / imported with CUDA IPC between two processes on one GPU."""
import ctypes
import os
import sys

import torch
import torch.distributed as dist



class Handle(ctypes.Structure):
    _fields_ = [("reserved", ctypes.c_char * 64)]


def main():
    dist.init_process_group("gloo")
    r = dist.get_rank()
    torch.cuda.set_device(0)
    rt = ctypes.CDLL("/usr/local/cuda/lib64/libcudart.so")
    sizes = [256, 4096, 1 << 20, 2 << 20, 32 << 20, 256 << 20, 1 << 30, 3 << 30]
    ptrs, hs = [], []
    for s in sizes:
        p = ctypes.c_void_p()
        assert rt.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(s)) == 0
        h = Handle()
        e = rt.cudaIpcGetMemHandle(ctypes.byref(h), p)
        ptrs.append(p)
        hs.append(bytes(h))
        print(r, "get", s, e, flush=True)
    allh = [None, None]
    dist.all_gather_object(allh, hs)
    if r == 1:
        for s, h in zip(sizes, allh[0]):
            q = ctypes.c_void_p()
            hb = Handle.from_buffer_copy(h)
            rt.cudaIpcOpenMemHandle.argtypes = [ctypes.POINTER(ctypes.c_void_p), Handle, ctypes.c_uint]
            e = rt.cudaIpcOpenMemHandle(ctypes.byref(q), hb, 1)
            print("open", s, e, flush=True)
    dist.barrier()


main()
