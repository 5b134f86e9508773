"""Experiment: fastest way to land a device buffer in a fresh Python bytes object."""
import ctypes, time, torch
n = 500 << 20
dev = torch.randint(0, 255, (n,), dtype=torch.uint8, device="cuda")
pin = torch.empty(n, dtype=torch.uint8, pin_memory=True)
api = ctypes.pythonapi
api.PyBytes_FromStringAndSize.restype = ctypes.py_object
api.PyBytes_FromStringAndSize.argtypes = [ctypes.c_void_p, ctypes.c_ssize_t]
libc = ctypes.CDLL("libc.so.6")
libc.madvise.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_int]
cudart = ctypes.CDLL(torch.cuda.__file__.rsplit("/", 1)[0] + "/../lib/libcudart.so.12") if False else None
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip(), open("/sys/kernel/mm/transparent_hugepage/defrag").read().strip())
def T(): torch.cuda.synchronize(); return time.perf_counter()
for rep in range(3):
    t0 = T(); pin.copy_(dev); b = pin.numpy().tobytes(); t1 = T()
    del b
    t2 = T(); b = api.PyBytes_FromStringAndSize(None, n); addr = ctypes.cast(ctypes.c_char_p(b), ctypes.c_void_p).value
    s = (addr + (2 << 20) - 1) & ~((2 << 20) - 1); e = (addr + n) & ~((2 << 20) - 1)
    r = libc.madvise(s, e - s, 14)
    pin.copy_(dev); ctypes.memmove(addr, pin.data_ptr(), n); t3 = T()
    del b
    t4 = T(); b = api.PyBytes_FromStringAndSize(None, n); addr = ctypes.cast(ctypes.c_char_p(b), ctypes.c_void_p).value
    ctypes.memmove(addr, pin.data_ptr(), n); t5 = T()
    del b
    t6 = T(); b = api.PyBytes_FromStringAndSize(None, n); addr = ctypes.cast(ctypes.c_char_p(b), ctypes.c_void_p).value
    cudaHostRegister = torch.cuda.cudart().cudaHostRegister
    rr = cudaHostRegister(addr, n, 0)
    h = torch.from_numpy(__import__("numpy").frombuffer((ctypes.c_ubyte * n).from_address(addr), dtype="u1"))
    h.copy_(dev)
    torch.cuda.cudart().cudaHostUnregister(addr); t7 = T()
    del b, h
    print(f"tobytes {t1-t0:.4f}  madvise(huge)+memmove {t3-t2:.4f} (rc {r})  plain memmove {t5-t4:.4f}  hostRegister+DMA {t7-t6:.4f} (rc {rr})")
