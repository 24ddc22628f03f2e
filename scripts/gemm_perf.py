import ctypes as C, torch, sys, json
sys.path.insert(0,'.')
from paper_2507_18006_b200 import _lib
lib=_lib.load()
res=[]
for (name,N,K) in [("qkv",12288,4096),("o",4096,4096),("gu",22016,4096),("down",4096,11008),("head",32000,4096)]:
    w=torch.randn(N,K,device='cuda').to(torch.bfloat16)
    for T in (1,16,64,128,256,2048,8192):
        x=torch.randn(T,K,device='cuda').to(torch.bfloat16)
        out=torch.empty(T,N,device='cuda',dtype=torch.bfloat16)
        ms=C.c_float()
        st=lib.cbt_gemm_bench(C.c_void_p(w.data_ptr()),C.c_void_p(x.data_ptr()),T,N,K,T,0,C.c_void_p(out.data_ptr()),N,20,C.byref(ms))
        assert st==0
        gbs=(N*K*2+T*K*2+T*N*2)/ms.value/1e6
        tf=2*N*K*T/ms.value/1e9
        res.append((name,N,K,T,round(ms.value*1000,1),round(gbs),round(tf,1)))
        print(name,N,K,T,f"{ms.value*1000:.1f}us {gbs:.0f} GB/s {tf:.1f} TF/s",flush=True)
