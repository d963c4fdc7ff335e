import torch, time
dev=torch.device('cuda',0)
nb=1<<30
h1=torch.empty(nb,dtype=torch.uint8).pin_memory(); h2=torch.empty(nb,dtype=torch.uint8).pin_memory()
d1=torch.empty(nb,dtype=torch.uint8,device=dev); d2=torch.empty(nb,dtype=torch.uint8,device=dev)
s1=torch.cuda.Stream(); s2=torch.cuda.Stream()
def run(fs, reps=5):
    for f in fs: f()
    torch.cuda.synchronize(); t=time.perf_counter()
    for _ in range(reps):
        for f in fs: f()
    torch.cuda.synchronize(); return (time.perf_counter()-t)/reps
def h2d():
    with torch.cuda.stream(s1): d1.copy_(h1,non_blocking=True)
def d2h():
    with torch.cuda.stream(s2): h2.copy_(d2,non_blocking=True)
t1=run([h2d]); t2=run([d2h]); t3=run([h2d,d2h])
print("h2d %.1f GB/s d2h %.1f GB/s duplex %.1f GB/s (each %.1f)"%(nb/t1/1e9, nb/t2/1e9, 2*nb/t3/1e9, nb/t3/1e9))
# chunked h2d 32MB pieces over 3 streams
ss=[torch.cuda.Stream() for _ in range(3)]
c=32<<20
def chunked():
    for i in range(nb//c):
        with torch.cuda.stream(ss[i%3]): d1[i*c:(i+1)*c].copy_(h1[i*c:(i+1)*c],non_blocking=True)
t4=run([chunked]); print("h2d chunked 32MB x3 streams %.1f GB/s"%(nb/t4/1e9))
