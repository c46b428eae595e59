import torch, sys
sys.path.insert(0,'.')
from paper_2506_19693_b200 import _native as nat
sink=torch.zeros(1,dtype=torch.int64,device='cuda')
sms=torch.cuda.get_device_properties(0).multi_processor_count
p40=1099511922689
for name,fn,p in (('int',nat.LIB.ckb_alu_probe,p40),('f64',nat.LIB.ckb_alu_probe_f64,p40)):
  for bm in (8,16,32):
    blocks,iters=sms*bm,400
    nat.check(fn(p,(2*p)//3,10,blocks,nat.ptr(sink),nat.stream_handle()),'p')
    a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); a.record()
    nat.check(fn(p,(2*p)//3,iters,blocks,nat.ptr(sink),nat.stream_handle()),'p')
    b.record(); torch.cuda.synchronize()
    print(name, bm, 'Gbfly/s', round(blocks*256*12*iters/(a.elapsed_time(b)/1e3)/1e9,1))
