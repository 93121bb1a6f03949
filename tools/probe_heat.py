"""Dev probe: tcgen05 heat map vs a numpy overlap oracle on random edge maps."""
import ctypes as C, sys, time
import numpy as np, torch
sys.path.insert(0, '.')
lib = C.CDLL('paper_2301_03047_b200/libglr_b200.so')
lib.glr_last_error.restype = C.c_char_p
def chk(st):
    if st != 0: raise RuntimeError(lib.glr_last_error().decode())

def heat_np(maps, anchors, P):
    # maps (4,H,W,C) u8
    H, W = maps.shape[1:3]
    E = np.concatenate(list(maps), axis=2).astype(np.int64)  # H,W,4C
    oh, ow = H-P+1, W-P+1
    out = np.zeros((len(anchors), oh, ow), np.int64)
    for n,(r,c) in enumerate(anchors):
        k = E[r:r+P, c:c+P, :]
        for p in range(P):
            for q in range(P):
                out[n] += (E[p:p+oh, q:q+ow, :] * k[p, q]).sum(-1)
    return out

def run(H, W, Cc, P, N, seed, dens=0.3):
    rng = np.random.default_rng(seed)
    maps = (rng.random((4, H, W, Cc)) < dens).astype(np.uint8)
    anchors = np.stack([rng.integers(0, H-P+1, N), rng.integers(0, W-P+1, N)], 1).astype(np.int32)
    e = lib.glr_heat_expand_factor(Cc, P)
    lib.glr_heat_workspace.restype = C.c_size_t
    ws_b = lib.glr_heat_workspace(Cc, P, N)
    dmaps = torch.from_numpy(maps).cuda()
    stack = torch.zeros(H*W*4*Cc*e, dtype=torch.uint8, device='cuda')
    chk(lib.glr_stack_from_maps(C.c_void_p(dmaps.data_ptr()), H, W, Cc, e, C.c_void_p(stack.data_ptr()), None))
    danc = torch.from_numpy(anchors).cuda()
    oh, ow = H-P+1, W-P+1
    lib.glr_heat_stride.restype = C.c_int64
    stride = lib.glr_heat_stride(H, W, P)
    heat = torch.zeros((N, stride), dtype=torch.int16, device='cuda')
    ws = torch.empty(ws_b, dtype=torch.uint8, device='cuda')
    lib.glr_heat_map.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_void_p]
    chk(lib.glr_heat_map(stack.data_ptr(), H, W, Cc, P, e, danc.data_ptr(), N, None, heat.data_ptr(), ws.data_ptr(), ws_b, None))
    torch.cuda.synchronize()
    got = heat.cpu().numpy().view(np.uint16)[:, :oh*ow].reshape(N, oh, ow).astype(np.int64)
    ref = heat_np(maps, anchors, P)
    ok = np.array_equal(got, ref)
    print(f"H={H} W={W} C={Cc} P={P} N={N} e={e}: {'OK' if ok else 'MISMATCH'}", flush=True)
    if not ok:
        d = np.argwhere(got != ref)
        print('  first diffs', d[:5], got[tuple(d[0])], ref[tuple(d[0])], 'ndiff', len(d))
    return ok

allok = True
for args in [(20, 18, 2, 6, 3, 0), (40, 37, 1, 8, 5, 1), (33, 150, 3, 4, 7, 2), (64, 64, 4, 8, 300, 3),
             (50, 140, 24, 8, 40, 4), (60, 61, 1, 12, 20, 5), (30, 30, 2, 8, 260, 6), (45, 47, 16, 8, 17, 7),
             (9, 9, 1, 3, 2, 8), (40, 200, 5, 5, 9, 9)]:
    allok &= run(*args)
# timing at the C2 shape
H=W=1024; Cc=24; P=8; N=4096
rng = np.random.default_rng(0)
e = lib.glr_heat_expand_factor(Cc, P)
stack = torch.from_numpy((rng.random(H*W*4*Cc*e) < 0.2).astype(np.uint8)).cuda()
anchors = torch.from_numpy(np.stack([rng.integers(0, H-P+1, N), rng.integers(0, W-P+1, N)], 1).astype(np.int32)).cuda()
ws_b = lib.glr_heat_workspace(Cc, P, N); ws = torch.empty(ws_b, dtype=torch.uint8, device='cuda')
lib.glr_heat_stride.restype = C.c_int64
heat = torch.empty((N, lib.glr_heat_stride(H, W, P)), dtype=torch.int16, device='cuda')
for it in range(4):
    s = torch.cuda.Event(enable_timing=True); t = torch.cuda.Event(enable_timing=True)
    s.record()
    chk(lib.glr_heat_map(stack.data_ptr(), H, W, Cc, P, e, anchors.data_ptr(), N, None, heat.data_ptr(), ws.data_ptr(), ws_b, None))
    t.record(); torch.cuda.synchronize()
    ms = s.elapsed_time(t)
    fl = 2.0*(H-P+1)*(W-P+1)*4*Cc*P*P*N
    print(f"C2 heat: {ms:.2f} ms  {fl/ms/1e9:.1f} TOPS", flush=True)
print("ALLOK" if allok else "FAIL")
