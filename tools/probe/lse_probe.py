import torch, math
B,S,H,hd=2,256,4,64
q,k,v=(torch.randn((B,S,H,hd),device="cuda",dtype=torch.bfloat16) for _ in range(3))
qt,kt,vt=(t.transpose(1,2) for t in (q,k,v))
r=torch.ops.aten._scaled_dot_product_cudnn_attention(qt,kt,vt,None,True,0.0,True,False)
print([type(x) if not torch.is_tensor(x) else (x.shape,x.dtype,x.stride()) for x in r])
o,lse=r[0],r[1]
s=(qt.float()@kt.float().transpose(-1,-2))/math.sqrt(hd)
mask=torch.triu(torch.ones(S,S,device="cuda",dtype=torch.bool),1)
s=s.masked_fill(mask,float("-inf"))
ref=torch.logsumexp(s,-1)
print("lse err natural", (lse.reshape(ref.shape)-ref).abs().max().item(), "log2", (lse.reshape(ref.shape)-ref/math.log(2)).abs().max().item())
print("o stride", o.stride())
