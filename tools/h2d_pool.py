import ctypes, glob, time, os, torch, numpy as np
import nvidia
cands = glob.glob(os.path.join(os.path.dirname(nvidia.__path__[0]), "nvidia", "cuda_runtime", "lib", "libcudart.so*"))
cands += glob.glob("/usr/local/cuda/lib64/libcudart.so*")
print(cands)
rt = ctypes.CDLL(cands[0])
torch.cuda.init()
n = 4 << 30
h = torch.empty(n, dtype=torch.uint8).pin_memory()
h.fill_(7)
def t_copy(dst, tag):
    for _ in range(3):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        assert rt.cudaMemcpy(ctypes.c_void_p(dst), ctypes.c_void_p(h.data_ptr()), ctypes.c_size_t(n), 1) == 0
        torch.cuda.synchronize(); print(tag, f"{1e3*(time.perf_counter()-t0):.1f} ms")
p = ctypes.c_void_p()
assert rt.cudaMalloc(ctypes.byref(p), ctypes.c_size_t(n)) == 0
t_copy(p.value, "cudaMalloc")
q = ctypes.c_void_p()
assert rt.cudaMallocAsync(ctypes.byref(q), ctypes.c_size_t(n), None) == 0
rt.cudaStreamSynchronize(None)
t_copy(q.value, "cudaMallocAsync")
x = torch.empty(n, dtype=torch.uint8, device="cuda")
t_copy(x.data_ptr(), "torch")
