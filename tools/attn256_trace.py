import ctypes as C, sys, json, torch
sys.path.insert(0, ".")
from paper_2310_16355_b200 import _lib
L=_lib.lib()
B,T,Hl,hd=4,2048,16,256
Dl=Hl*hd
g=torch.Generator(device="cuda").manual_seed(0)
qkv=torch.randn(B*T,3*Dl,generator=g,device="cuda").bfloat16()
o=torch.empty(B*T,Dl,device="cuda",dtype=torch.bfloat16); lse=torch.empty(B,Hl,T,device="cuda")
dout=torch.randn(B*T,Dl,generator=g,device="cuda").bfloat16(); dqkv=torch.empty_like(qkv)
scr=torch.empty(B*T*Hl+B*T*2*Dl,device="cuda")
L.sw_k_attention_fwd(qkv.data_ptr(),o.data_ptr(),lse.data_ptr(),B,T,Hl,hd,None)
for _ in range(3):
    L.sw_k_attention_bwd(qkv.data_ptr(),o.data_ptr(),lse.data_ptr(),dout.data_ptr(),dqkv.data_ptr(),scr.data_ptr(),B,T,Hl,hd,None)
torch.cuda.synchronize()
buf=(C.c_ulonglong*4096)()
L.sw_k_attention_trace.argtypes=[C.c_void_p]
L.sw_k_attention_trace(buf)
t0=buf[0]
for n in range(34):
    b=[buf[16*n+i] for i in range(10)]
    if b[0]==0: break
    print(n, [int(x-t0) if x else None for x in b])
