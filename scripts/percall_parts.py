"""Where a per-call walk's time goes (not part of the product): the ctypes
call of pv_server_walk alone, cudaStreamQuery alone, the PerCall.walk wrapper
and the public translate, each timed over n calls on the box."""
import ctypes
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def per_call(fn, n=5000):
    for _ in range(500):
        fn()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    return (time.perf_counter() - t0) / n * 1e6


def main():
    import torch

    from paper_1304_3771_b200 import _native as N
    from paper_1304_3771_b200 import percall
    from paper_1304_3771_b200 import workloads as W

    memv, guest, space = W.build_c1("shadow", device=True)
    tr = memv.translator(space, use_cache=False)
    img = memv.host_mem.backing
    sp = tr.device_space
    pc = percall.get()
    lib = N.lib()
    dev = img.device()
    ptr, nb = dev.data_ptr(), img.nbytes
    s = torch.cuda.current_stream().cuda_stream
    va = W.C1_GVA + 0x1234
    pc.walk(img, sp, va, False)
    out = {}
    out["ctypes pv_server_walk"] = per_call(lambda: lib.pv_server_walk(ptr, nb, pc.space_ref, va, 0, pc.one_ptr, s))
    rt = ctypes.CDLL("libcudart.so.12") if False else None
    try:
        rt = ctypes.CDLL(os.path.join(os.path.dirname(torch.__file__), "lib", "libcudart.so.12"))
    except OSError:
        import glob
        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia", "cuda_runtime", "lib",
                                       "libcudart.so*"))
        rt = ctypes.CDLL(cands[0]) if cands else None
    if rt is not None:
        rt.cudaStreamQuery.argtypes = [ctypes.c_void_p]
        out["ctypes cudaStreamQuery"] = per_call(lambda: rt.cudaStreamQuery(s))
    out["ctypes pv_abi_version (ctypes floor)"] = per_call(lambda: lib.pv_abi_version())
    out["PerCall.walk"] = per_call(lambda: pc.walk(img, sp, va, False))
    out["ProcessTranslator.translate"] = per_call(lambda: tr.translate(va))
    percall.park()
    percall._SERVER = False
    out["PerCall.walk (launch per call)"] = per_call(lambda: pc.walk(img, sp, va, False))
    print(json.dumps({k: round(v, 2) for k, v in out.items()}, indent=1))


if __name__ == "__main__":
    main()
