import sys, math, torch
sys.path.insert(0, '.')
from paper_2311_18677_b200 import kernels as K
torch.manual_seed(0)
H=Hkv=32; dh=128; bs=16; ctx=[1,17,300,1100]; B=4; maxb=80; nblk=400
kp=torch.randn(nblk,Hkv,bs,dh,device='cuda').bfloat16(); vp=torch.randn_like(kp)
tables=torch.randperm(nblk,device='cuda').int()[:B*maxb].view(B,maxb).contiguous()
qkv=torch.randn(B,(H+2*Hkv)*dh,device='cuda').bfloat16()
lens=torch.tensor(ctx,device='cuda',dtype=torch.int32)
for part in (256,128):
  ws=torch.zeros(K.attn_decode_workspace_bytes(B,H,1200,part,dh),dtype=torch.uint8,device='cuda')
  outs=[K.attn_decode(qkv,kp.data_ptr(),vp.data_ptr(),tables,lens,B,H,Hkv,dh,bs,1/math.sqrt(dh),1200,part,ws).clone() for _ in range(4)]
  torch.cuda.synchronize()
  for i in range(1,4):
    d=(outs[i].float()-outs[0].float()).abs().view(B,H,dh)
    print(part, i, d.max().item(), [(b, d[b].max().item()) for b in range(B)])
  np_=(1200+part-1)//part
  t=ws[B*H*np_*(dh+2)*4:].view(torch.int32)
  print('tickets', t[:B*Hkv].tolist()[:8])
