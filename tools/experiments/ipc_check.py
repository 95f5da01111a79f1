import torch, torch.multiprocessing as mp, time, subprocess
def child(q, done):
    t = q.get()
    t.add_(1.0)
    torch.cuda.synchronize()
    done.put(float(t.sum().item()))
if __name__ == "__main__":
    print(subprocess.run(["nvidia-smi","--query-gpu=compute_mode,name","--format=csv"],capture_output=True,text=True).stdout)
    mp.set_start_method("spawn")
    q, done = mp.Queue(), mp.Queue()
    p = mp.Process(target=child, args=(q, done)); p.start()
    t = torch.zeros(1024, device="cuda:0"); q.put(t)
    print("child sum", done.get(timeout=120)); p.join()
    torch.cuda.synchronize(); print("parent sees", float(t.sum().item()))
