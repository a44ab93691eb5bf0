import torch, json
def t(fn, n=50):
    for _ in range(5): fn()
    torch.cuda.synchronize()
    e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1)/n*1e3
for M,N,K in [(3072,768,8192),(768,3072,8192),(2304,768,8192),(768,768,8192),(4096,4096,8192),(8192,8192,8192)]:
    dy=torch.randn(K,M,device='cuda',dtype=torch.bfloat16); x=torch.randn(K,N,device='cuda',dtype=torch.bfloat16)
    a=torch.randn(M,K,device='cuda',dtype=torch.bfloat16); b=torch.randn(N,K,device='cuda',dtype=torch.bfloat16)
    f=2*M*N*K
    r={}
    for name,fn in [('mn_major_f32out',lambda: torch.mm(dy.t(),x,out_dtype=torch.float32)),('k_major_f32out',lambda: torch.mm(a,b.t(),out_dtype=torch.float32)),('mn_major_bf16',lambda: torch.mm(dy.t(),x)),('k_major_bf16',lambda: torch.mm(a,b.t()))]:
        us=t(fn); r[name]=round(f/us/1e6,1)
    print(json.dumps({"MNK":[M,N,K],"tflops":r}))
