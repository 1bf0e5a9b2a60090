"""Zero-copy dropout: the fused kernel reads x from and writes y to pinned host memory
directly over PCIe (UVA), vs the staged 3-stream pipeline."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2509_07003_b200 import _lib, ops, rng as R
from paper_2509_07003_b200.rng import dtype_code
from paper_2509_07003_b200.placement import full_view
shape = (8, 4096, 4096)
xh = torch.randn(shape, dtype=torch.bfloat16).pin_memory(); yh = torch.empty_like(xh).pin_memory()
st = R.RngState(20240817); view = full_view(shape)
def zc():
    nr, nv = st.native(), view.to_native()
    s = _lib.LIB.sdr_dropout(xh.data_ptr(), dtype_code(xh.dtype), yh.data_ptr(), dtype_code(xh.dtype), None, -1, 0.1,
                             C.byref(nr), C.byref(nv), _lib.stream_handle(torch.device("cuda", 0)))
    assert s == 0, s
    torch.cuda.current_stream().synchronize()
for name, fn in [("zero-copy", zc), ("staged", lambda: ops.dropout_host(xh, 0.1, st, out=yh))]:
    fn()
    t0 = time.perf_counter()
    for _ in range(5): fn()
    dt = (time.perf_counter() - t0) / 5
    print(f"{name}: {dt*1e3:.2f} ms  {xh.numel()*4/dt/1e9:.1f} GB/s", flush=True)
ref = ops.dropout_apply(xh.cuda(), 0.1, st).cpu()
zc()
print("zero-copy bit-exact vs device:", torch.equal(ref.view(torch.int16), yh.view(torch.int16)))
