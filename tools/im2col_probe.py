import sys, torch
sys.path.insert(0, '.')
from paper_2003_06795_b200 import conv
x = torch.rand((8, 64, 224, 224), device='cuda')
xb = x.bfloat16()
for _ in range(2):
    conv.im2col(x, 3, 3, 1, 1, family='f32')
    conv.im2col(xb, 3, 3, 1, 1, family='bf16')
torch.cuda.synchronize()
