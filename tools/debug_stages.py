import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1912_02165_b200 as wf
from paper_1912_02165_b200 import _lib, device as D
import torch

rng = np.random.default_rng(0)
spec = wf.LayerSpec(1, 16, 16, 8, 8, 3, 1, 1)
T = 4
x = rng.standard_normal(spec.input_dims()).astype(np.float32)
w = rng.standard_normal(spec.kernel_dims()).astype(np.float32)
basis = wf.make_basis(T)
pack = wf.transform_kernels(wf.Tensor4D(w), basis)
pl = wf.tile_plan(spec, T)
# numpy U (T^2, n_tile, C)
U = np.zeros((T*T, pl.n_tile, spec.in_channels), np.float32)
for i in range(pl.n_tile):
    c = pl.coord(i)
    for ch in range(spec.in_channels):
        win = wf.gather_input_tile(wf.Tensor4D(x), pl, c, ch)
        U[:, i, ch] = (basis.bt32 @ win @ basis.bt32.T).reshape(-1)
M = np.einsum("pnc,pcd->pnd", U.astype(np.float64), pack.data.astype(np.float64))
dev = torch.device("cuda", 0)
lib = _lib.load()
layer = _lib.layer_struct(spec)
need = lib.wf_three_stage_scratch_bytes(layer, T, 0)
scratch = torch.zeros(need, dtype=torch.uint8, device=dev)
xd = D.to_device(x, dev); y = torch.empty(spec.output_dims(), device=dev)
vp = pack.device_mma(dev)
_lib.check(lib.wf_conv_three_stage(D.ptr(xd), D.ptr(vp), D.ptr(y), D.ptr(scratch), need, layer, T, 0, 0, D.stream_ptr(dev)), "3s")
torch.cuda.synchronize()
sc = scratch.cpu().numpy()
Cpad = 16; nblk = 1; slab = 128 * Cpad * 2
def slab_off(row, k, rows, Kpad):
    j, kk = k >> 6, k & 63
    kc = min(64, Kpad - 64 * j)
    return j * rows * 128 + (row >> 3) * (16 * kc) + (kk >> 3) * 128 + (row & 7) * 16 + (kk & 7) * 2
def bf(raw):  # uint16 -> float
    return (raw.astype(np.uint32) << 16).view(np.float32)
Ug = np.zeros_like(U)
for p in range(T*T):
    for n in range(pl.n_tile):
        for ch in range(spec.in_channels):
            o = slab_off(n, ch, 128, Cpad)
            hi = sc[p*2*slab + o: p*2*slab + o + 2].view(np.uint16)
            lo = sc[p*2*slab + slab + o: p*2*slab + slab + o + 2].view(np.uint16)
            Ug[p, n, ch] = bf(hi)[0] + bf(lo)[0]
print("U max abs err", np.abs(Ug - U).max(), "max U", np.abs(U).max())
Moff = T*T*nblk*2*slab
Mg = sc[Moff:Moff + T*T*spec.out_channels*128*4].view(np.float32).reshape(T*T, spec.out_channels, 128)[:, :, :pl.n_tile].transpose(0, 2, 1)
print("M max abs err", np.abs(Mg - M).max(), "max M", np.abs(M).max())
print("M sample got", Mg[0, 0, :4], "want", M[0, 0, :4])
# V check: decode mma pack
vpk = vp.cpu().numpy(); vslab = 16 * 16 * 2
V = np.zeros((T*T, 16, 16), np.float32)
for p in range(T*T):
    for n in range(16):
        for k in range(16):
            o = slab_off(n, k, 16, 16)
            V[p, k, n] = bf(vpk[p*2*vslab+o:p*2*vslab+o+2].view(np.uint16))[0] + bf(vpk[p*2*vslab+vslab+o:p*2*vslab+vslab+o+2].view(np.uint16))[0]
print("V max abs err", np.abs(V - pack.data).max())
Mu = np.einsum("pnc,pcd->pnd", Ug.astype(np.float64), V.astype(np.float64))
print("M vs decoded-operand product", np.abs(Mg - Mu).max())
print("ratio sample", (Mg[0,:4,:4] / Mu[0,:4,:4]))
yg = y.cpu().numpy()
Y = np.zeros(spec.output_dims())
for i in range(pl.n_tile):
    c = pl.coord(i)
    for cp in range(spec.out_channels):
        blk = basis.at @ M[:, i, cp].reshape(T, T) @ basis.at.T
        oy, ox = pl.output_origin(c)
        ny = min(pl.out, spec.out_height - oy); nx = min(pl.out, spec.out_width - ox)
        Y[c.batch, cp, oy:oy+ny, ox:ox+nx] = blk[:ny, :nx]
print("Y (numpy from M) vs gpu", np.abs(Y - yg).max(), np.abs(Y).max())
xp = np.pad(x.astype(np.float64), ((0,0),(0,0),(1,1),(1,1)))
R = np.zeros(spec.output_dims())
for ky in range(3):
    for kx in range(3):
        R += np.einsum("bcyx,oc->boyx", xp[:, :, ky:ky+spec.out_height, kx:kx+spec.out_width], w[:, :, ky, kx].astype(np.float64))
print("Y(numpy) vs direct", np.abs(Y - R).max())
print(yg[0,0,:2,:4]); print(Y[0,0,:2,:4])
