import torch, torch.multiprocessing as mp
def child(q, r):
    t = q.get()
    t += 1
    torch.cuda.synchronize()
    r.put(float(t.sum().item()))
if __name__ == "__main__":
    mp.set_start_method("spawn")
    q, r = mp.Queue(), mp.Queue()
    p = mp.Process(target=child, args=(q, r)); p.start()
    t = torch.zeros(1024, device="cuda")
    q.put(t)
    print("child saw", r.get(timeout=60)); p.join()
    torch.cuda.synchronize()
    print("parent sees", float(t.sum().item()))
