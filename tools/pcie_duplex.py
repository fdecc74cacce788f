"""PCIe check: H2D and D2H of the C3 e2e sizes, alone and concurrently (pinned)."""
import torch
n_in, n_out = 78224356 // 4, 68446312 // 4
hi = torch.empty(n_in).pin_memory(); ho = torch.empty(n_out).pin_memory()
di = torch.empty(n_in, device="cuda"); do = torch.empty(n_out, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn):
    for _ in range(3): fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize(); return e0.elapsed_time(e1)
def h2d():
    s1.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1): di.copy_(hi, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
def d2h():
    s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)
def both():
    s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s1): di.copy_(hi, non_blocking=True)
    with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
print("h2d ms", t(h2d), "d2h ms", t(d2h), "both ms", t(both))
# chunked: H2D in K pieces on s1; D2H piece j on s2 after H2D piece j+1
for K in (2, 8):
    ev = [torch.cuda.Event() for _ in range(K)]
    def chunked():
        s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
        bi, bo = n_in // K, n_out // K
        with torch.cuda.stream(s1):
            for j in range(K):
                di[j * bi:(j + 1) * bi].copy_(hi[j * bi:(j + 1) * bi], non_blocking=True); ev[j].record(s1)
        with torch.cuda.stream(s2):
            for j in range(K):
                s2.wait_event(ev[min(j + 1, K - 1)])
                ho[j * bo:(j + 1) * bo].copy_(do[j * bo:(j + 1) * bo], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    print("chunked", K, "ms", t(chunked))
