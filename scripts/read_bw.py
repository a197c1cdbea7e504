import torch, numpy as np
def t(fn, reps=20):
    for _ in range(3): fn()
    ts=[]
    for _ in range(reps):
        a,b=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
        a.record(); fn(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b)*1000)
    return float(np.median(ts))
x=torch.rand((410236,96),device='cuda'); w=torch.rand((96,16),device='cuda')
print('sum(1)', t(lambda: x.sum(1)), 'sum(0)', t(lambda: x.sum(0)), 'clone', t(lambda: x.clone()), 'mm', t(lambda: x@w))
y=torch.rand(410236*96*8,device='cuda')
print('big clone 1.26GB x2', t(lambda: y.clone()))
