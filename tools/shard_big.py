import sys, os, numpy as np, torch
sys.path.insert(0, '.')
from paper_1409_5757_b200 import _native
n = 1 << 30; G = 8
x = torch.randn(n, dtype=torch.complex64, device='cuda')
p1 = _native.NativePlan(n, _native.EFFT_C64, -1, 0); y = torch.empty_like(x)
s = torch.cuda.current_stream().cuda_stream
p1.execute(x.data_ptr(), y.data_ptr(), s); torch.cuda.synchronize()
del p1
for chunks in ("1", "4"):
    os.environ["EFFT_SHARD_CHUNKS"] = chunks
    plan = _native.ShardedPlan(n, _native.EFFT_C64, -1, [0] * G)
    d_in = list(torch.chunk(x, G)); d_out = [torch.empty_like(t) for t in d_in]
    streams = [torch.cuda.Stream() for _ in range(G)]
    torch.cuda.synchronize()
    for rep in range(2):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        plan.execute([t.data_ptr() for t in d_in], [t.data_ptr() for t in d_out], [st.cuda_stream for st in streams])
        torch.cuda.synchronize(); e1.record(); torch.cuda.synchronize()
    z = torch.cat(d_out)
    err = (torch.linalg.vector_norm((z - y).to(torch.complex128)) / torch.linalg.vector_norm(y.to(torch.complex128))).item()
    print(f"sharded G={G} chunks={chunks}: rel-L2 vs single-GPU {err:.3e}, {e0.elapsed_time(e1):.1f} ms (8 emulated ranks on one GPU)")
    del plan, d_out, z
