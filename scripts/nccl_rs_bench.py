"""Isolated NCCL ReduceScatter / AllGather timing at the RN50 plan's chunk sizes (torchrun, N ranks):
ncclAvg vs ncclSum (NVLS reduces in the switch for sum), to size the RS / AG stages of bench.py."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import paper_1811_12019_b200 as K  # noqa: E402
from synth import shapes  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(rank)
dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
layers, n = shapes.config("resnet50")
q = K.Plan(layers, world, n, K.LPT).query()
for name, chunk in (("rs", q["rs_chunk"]), ("ag", q["ag_chunk"])):
    send = torch.randn(world * chunk, device=dev)
    recv = torch.empty(chunk, device=dev)
    for op_name, op in (("sum", dist.ReduceOp.SUM), ("avg", dist.ReduceOp.AVG)):
        if name == "ag" and op_name == "avg":
            continue
        for _ in range(3):
            dist.reduce_scatter_tensor(recv, send, op=op) if name == "rs" else dist.all_gather_into_tensor(send, recv)
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20):
            dist.reduce_scatter_tensor(recv, send, op=op) if name == "rs" else dist.all_gather_into_tensor(send, recv)
        e1.record()
        torch.cuda.synchronize()
        ms = torch.tensor([e0.elapsed_time(e1) / 20], device=dev)
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
        busbw = chunk * 4 * (world - 1) / (ms.item() / 1e3) / 1e9
        if rank == 0:
            print(f"{name} {op_name} P={world} chunk {chunk * 4 / 1e6:.1f} MB: {ms.item():.3f} ms, bus {busbw:.0f} GB/s", flush=True)
dist.destroy_process_group()
