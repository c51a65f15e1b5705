"""Per-rank cost of the regular vs the exchange form of a C4 slab (KB kernel time
via ctx profiling, whole call via events) and the device merge of 8 slabs' maxima."""
import sys, os, ctypes as C, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_1310_6736_b200 import _lib, api, sharding
from paper_1310_6736_b200._lib import Context
from tests import phantoms
SCALES=[float(s) for s in range(3,16)]
ctx=Context(0); dev=torch.device('cuda',0); st=torch.cuda.current_stream(dev); ctx.set_stream(st.cuda_stream)
vol,_=api.make_phantom(phantoms.config_c4()); nz,ny,nx=vol.shape
d_vol=torch.from_numpy(vol).to(dev); sc=np.asarray(SCALES); iw=_lib.Window(0.0,32.0,32,0); R=sharding.halo_radius(SCALES)
for world in (2,8):
  z0,z1,zs0,zs1=sharding.slab_bounds(nz,world,0 if world==2 else 3,R)
  d_slab=d_vol[zs0:zs1].contiguous(); d_score=torch.empty((z1-z0,ny,nx),device=dev); d_best=torch.empty_like(d_score); n=C.c_int64(0)
  def reg():
    _lib.check(_lib.load().salvox_exhaustive_slab_device(ctx.handle,C.c_void_p(d_slab.data_ptr()),nx,ny,nz,zs0,zs1,z0,z1,C.byref(iw),sc.ctypes.data_as(C.c_void_p),len(sc),0,10**15,C.c_void_p(d_score.data_ptr()),C.c_void_p(d_best.data_ptr()),C.byref(n)))
  def exch():
    api.exhaustive_slab_scores(d_slab,nz,zs0,z0,z1,SCALES,0.0,32.0,32,budget=10**15,ctx=ctx,out=(d_score,d_best))
    api.exhaustive_slab_maxima(d_vol[z0-1].contiguous() if z0>0 else None, d_vol[min(z1,nz-1)].contiguous() if z1<nz else None, ctx=ctx)
  for name,f in (('reg',reg),('exch',exch),('reg',reg),('exch',exch)):
    f(); torch.cuda.synchronize()
    ctx.set_profiling(True)
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record(st); f(); e1.record(st); e1.synchronize()
    kb=ctx.kernel_time(); ctx.set_profiling(False)
    print(world, name, 'total', round(e0.elapsed_time(e1),2), 'kb', round(kb[0],2), kb[1], kb[2])
# device merge cost at the N=8 size: 8 slabs' maxima (this slab's list 8 times, indices shifted)
z0,z1,zs0,zs1=sharding.slab_bounds(nz,8,3,R)
d_slab=d_vol[zs0:zs1].contiguous(); d_score=torch.empty((z1-z0,ny,nx),device=dev); d_best=torch.empty_like(d_score)
api.exhaustive_slab_scores(d_slab,nz,zs0,z0,z1,SCALES,0.0,32.0,32,budget=10**15,ctx=ctx,out=(d_score,d_best))
n = api.exhaustive_slab_maxima(d_vol[z0-1].contiguous(), d_vol[z1].contiguous(), ctx=ctx, on_device=True)
buf = torch.zeros((n, 48), dtype=torch.uint8, device=dev)
api.last_maxima_device(buf, ctx=ctx)
parts=[]
for r in range(8):
    p = buf.clone().view(torch.int64)
    p[:, 5] += r * nx * ny * 64
    parts.append(p.view(torch.uint8))
cat = torch.cat(parts)
api.merge_maxima_device(cat, ctx=ctx); torch.cuda.synchronize()
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
e0.record(st); out = api.merge_maxima_device(cat, ctx=ctx); e1.record(st); e1.synchronize()
print('maxima per slab', n, 'merge of', cat.shape[0], 'records ms', round(e0.elapsed_time(e1), 3))
