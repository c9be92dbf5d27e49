import cProfile, pstats, os, sys, io
sys.path.insert(0, '.')
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29633")
import torch, torch.distributed as dist
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
import paper_2505_00136_b200 as gpb
from paper_2505_00136_b200.distributed import DistributedGP
train, test = gpb.make_msd_dataset(65536, 256, 8, seed=0)
rt = gpb.start_runtime()
m = DistributedGP(train, gpb.KernelParams(), 128); m.log_likelihood(); m.close()
m = DistributedGP(train, gpb.KernelParams(), 128)
pr = cProfile.Profile(); pr.enable(); m._factor(); pr.disable()
print("enqueue", m.timings["enqueue_ms"])
st = io.StringIO(); pstats.Stats(pr, stream=st).sort_stats("tottime").print_stats(18); print(st.getvalue()[:6000])
rt.stop()
