import torch, paper_1712_02616_b200 as iabn
x = torch.randn(16, 4096, 112 * 112, device="cuda", dtype=torch.bfloat16)
g, b = torch.ones(4096, device="cuda"), torch.zeros(4096, device="cuda")
z, mean, var = iabn.forward(x, g, b)                 # z is x, overwritten
dx, dg, db = iabn.backward(z, torch.randn_like(z), g, b, var)   # dx over dz
layer = iabn.InPlaceABN(256, activation="sigmoid", device="cuda")  # fp32
y = layer(torch.randn(8, 256, 28, 28, device="cuda") * 1.0)        # autograd: z over x
y.sum().backward()
torch.cuda.synchronize()
print("readme ok", tuple(y.shape), float(y.min()), float(y.max()), layer.weight.grad.abs().sum().item() > 0)
