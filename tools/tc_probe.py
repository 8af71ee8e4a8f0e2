import ctypes, subprocess, sys, numpy as np, torch
subprocess.check_call("nvcc -gencode arch=compute_100a,code=sm_100a -O2 -shared -Xcompiler -fPIC -o /tmp/tcp.so tools/tc_probe.cu", shell=True)
L = ctypes.CDLL("/tmp/tcp.so")
L.run_probe.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_ulonglong, ctypes.c_uint]
dev = torch.device("cuda:0")
def run(mode, A, B, dx=0, ix=0):
    tA, tB = torch.from_numpy(A).to(dev), torch.from_numpy(B).to(dev)
    out = torch.full((128, 128), -7.0, device=dev); info = torch.zeros(4, dtype=torch.int32, device=dev)
    rc = L.run_probe(mode, tA.data_ptr(), tB.data_ptr(), out.data_ptr(), info.data_ptr(), dx, ix)
    return rc, out.cpu().numpy(), info.cpu().numpy()
A = np.zeros((8, 128), np.float32); B = np.zeros((8, 128), np.float32)
rc, o, inf = run(0, A, B)
exp = np.arange(128)[:, None] * 1000 + np.arange(128)[None, :]
print("mode0 rc", rc, "tmem", hex(int(inf[0]) & 0xffffffff), "stld ok", np.array_equal(o, exp), o[:2, :4])
rng = np.random.default_rng(0)
A = rng.integers(-3, 4, (8, 128)).astype(np.float32); B = rng.integers(-3, 4, (8, 128)).astype(np.float32)
ref = A.T @ B
rc, o, inf = run(1, A, B)
print("mode1 rc", rc, "maxerr", np.abs(o - ref).max(), "nz", np.count_nonzero(o), o[:3, :4], ref[:3, :4])
# try swapped LBO/SBO
lbo, sbo = 256, 8
dx = (lbo << 16) ^ (sbo << 16) ^ (sbo << 32) ^ (lbo << 32)
rc, o, inf = run(1, A, B, dx=dx)
print("swap rc", rc, "maxerr", np.abs(o - ref).max(), "nz", np.count_nonzero(o))
# try K-major flags (bits 15,16 cleared)
rc, o, inf = run(1, A, B, ix=(1 << 15) | (1 << 16))  # MN flags on K-major data
print("kmaj rc", rc, "maxerr", np.abs(o - ref).max(), "nz", np.count_nonzero(o))
for name, cand in [("ref", ref), ("refT", ref.T)]:
    pass
