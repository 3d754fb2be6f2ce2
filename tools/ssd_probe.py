"""SSD roofline for the f3 store's access pattern: O_DIRECT reads of whole
block records (the payload S of one cache entry) at random record offsets of a
base segment, at several queue depths (threads), against one large sequential
stream.  python tools/ssd_probe.py BASE_SEGMENT RECORD_BYTES"""
import mmap
import os
import random
import sys
import threading
import time

path, S = sys.argv[1], int(sys.argv[2])
if len(sys.argv) > 3:  # create a test file of that many GiB (incompressible data, O_DIRECT)
    gib = int(sys.argv[3])
    buf = mmap.mmap(-1, 16 << 20)
    buf.write(os.urandom(16 << 20))
    wfd = os.open(path, os.O_WRONLY | os.O_CREAT | os.O_TRUNC | os.O_DIRECT, 0o644)
    t = time.perf_counter()
    for i in range(gib * 64):
        os.pwritev(wfd, [buf], i * (16 << 20))
    os.fsync(wfd)
    os.close(wfd)
    print(f"created {gib} GiB: sequential O_DIRECT write {gib * 2**30 / (time.perf_counter() - t) / 1e9:.2f} GB/s")
size = os.path.getsize(path)
n_rec = (size - 4096) // S
fd = os.open(path, os.O_RDONLY | os.O_DIRECT)


PINNED = []


def pinned(n):
    """page-aligned pinned (cudaHostAlloc) buffer, as the store's cache entries are"""
    import ctypes
    import torch
    t = torch.empty(n + 4096, dtype=torch.uint8).pin_memory()
    PINNED.append(t)
    a = (t.data_ptr() + 4095) // 4096 * 4096
    return (ctypes.c_char * n).from_address(a)


def run(qd, n_reads, seq=False, req=S, pin=False, seed=0):
    rng = random.Random(seed * 1000 + qd)
    offs = [4096 + i * req for i in range(n_reads)] if seq else \
        [4096 + rng.randrange(n_rec) * S for _ in range(n_reads)]
    bufs = [pinned(req) if pin else mmap.mmap(-1, req) for _ in range(qd)]
    nxt = [0]
    lock = threading.Lock()

    def work(b):
        while True:
            with lock:
                i = nxt[0]
                nxt[0] += 1
            if i >= len(offs):
                return
            os.preadv(fd, [b], offs[i])

    th = [threading.Thread(target=work, args=(bufs[q],)) for q in range(qd)]
    t = time.perf_counter()
    for x in th:
        x.start()
    for x in th:
        x.join()
    dt = time.perf_counter() - t
    return len(offs) * req / dt / 1e9


print(f"records {n_rec} x {S} B ({size / 2**30:.1f} GiB file)")
print(f"sequential 16 MiB QD1: {run(1, 256, True, 16 << 20):.2f} GB/s")
for pin in (False, True):
    for qd in (1, 4, 8, 16):
        print(f"random records QD{qd} {'pinned' if pin else 'pageable'}: "
              f"{run(qd, 600, pin=pin, seed=qd + 10 * pin):.2f} GB/s")
