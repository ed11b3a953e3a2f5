"""Probe: can two processes on one GPU pin (cudaHostRegister) the same / overlapping / disjoint
ranges of one tmpfs file?  Runs each case in two concurrent child processes."""
import ctypes as C
import mmap
import multiprocessing as mp
import os
import sys
import time

MiB = 1 << 20


def child(path, lo, hi, q, hold):
    import torch  # noqa: F401  (CUDA runtime init)
    rt = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
    if rt is None:
        import glob
        cands = glob.glob("/usr/local/cuda*/lib64/libcudart.so*")
        rt = C.CDLL(cands[0])
    rt.cudaSetDevice(0)
    fd = os.open(path, os.O_RDONLY)
    m = mmap.mmap(fd, hi - lo, mmap.MAP_SHARED, mmap.PROT_READ, offset=lo)
    addr = C.c_void_p.from_buffer_copy(C.c_size_t(C.addressof(C.c_char.from_buffer_copy(b"x"))))
    buf = (C.c_char * (hi - lo)).from_buffer(m) if False else None
    # address of the mapping
    ptr = C.c_void_p()
    libc = C.CDLL("libc.so.6")
    libc.mmap.restype = C.c_void_p
    libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
    p = libc.mmap(None, hi - lo, 1, 1 | 0x8000, fd, lo)  # PROT_READ, MAP_SHARED|MAP_POPULATE
    flags = 0x08 | 0x01 | 0x02  # ReadOnly | Portable | Mapped
    e = rt.cudaHostRegister(C.c_void_p(p), C.c_size_t(hi - lo), flags)
    q.put((os.getpid(), lo, hi, e))
    time.sleep(hold)
    rt.cudaHostUnregister(C.c_void_p(p))


def main():
    path = sys.argv[1] if len(sys.argv) > 1 else "/dev/shm/probe_register.bin"
    size = 256 * MiB
    if not os.path.exists(path) or os.path.getsize(path) != size:
        with open(path, "wb") as f:
            f.write(os.urandom(1 << 20) * (size >> 20))
    ctx = mp.get_context("spawn")
    for name, ranges in (("disjoint", [(0, 128 * MiB), (128 * MiB, 256 * MiB)]),
                         ("overlap", [(0, 144 * MiB), (128 * MiB, 256 * MiB)]),
                         ("same", [(0, 128 * MiB), (0, 128 * MiB)])):
        q = ctx.Queue()
        ps = [ctx.Process(target=child, args=(path, lo, hi, q, 4)) for lo, hi in ranges]
        for pr in ps:
            pr.start()
            time.sleep(1.5)
        for pr in ps:
            pr.join()
        res = [q.get() for _ in ps]
        print(name, [(r[1] >> 20, r[2] >> 20, r[3]) for r in res], flush=True)


if __name__ == "__main__":
    main()
