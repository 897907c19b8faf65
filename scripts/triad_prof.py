import torch
n = 1 << 28
a = torch.rand(n, device="cuda"); b = torch.rand(n, device="cuda"); c = torch.empty(n, device="cuda")
for _ in range(5):
    torch.add(a, b, out=c)
    a.add_(b, alpha=-0.1)
torch.cuda.synchronize()
