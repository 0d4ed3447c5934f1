import subprocess, threading, time, torch
dev = torch.device("cuda", 0)
a = torch.empty(1 << 28, dtype=torch.float64, device=dev)   # 2 GiB
b = torch.empty_like(a)
samples = []
stop = False
def sampler():
    while not stop:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_throttle_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        samples.append(out)
        time.sleep(0.2)
th = threading.Thread(target=sampler); th.start()
torch.cuda.synchronize()
t0 = time.time(); n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < 6:
    for _ in range(20): b.copy_(a)
    torch.cuda.synchronize(); n += 20
e1.record(); torch.cuda.synchronize()
stop = True; th.join()
ms = e0.elapsed_time(e1)
print("copy GB/s", round(n * 2 * a.numel() * 8 / (ms * 1e-3) / 1e9, 1))
print("\n".join(samples[5:-2:3]))
