"""Token-sharded data parallelism of the INT4 linear.

One process per GPU.  Rank r owns tokens [r * N_r, (r + 1) * N_r) of the global
batch: X and grad_Y are sharded on the token dimension N (the
linear sees N = S T tokens), W is replicated.  The forward and grad_X are
local; the only exchange is the sum of the per-shard grad_W partials.

LSS under sharding: each shard samples with its own budget N_r and its own
per-shard amax, so each shard's grad_W is an unbiased estimate of its own
share and their sum is unbiased for the whole batch.  Philox counters use the
global token index (token_offset = r * N_r), so the random streams do not
depend on how the batch is split (reading Z-20).

This module is plumbing only (process groups, offsets, the all-reduce); every
arithmetic step runs in the library's kernels.
"""
import os

import torch
import torch.distributed as dist


def env_world():
    """(rank, world_size, local_rank) from the torchrun environment."""
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend="nccl", device=None):
    """Initialise the default process group if WORLD_SIZE > 1 (127.0.0.1 rendezvous)."""
    rank, world, _ = env_world()
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
        dist.init_process_group(backend, rank=rank, world_size=world, **kw)
    return rank, world


def token_offset(rank, tokens_per_rank):
    """Global index of this shard's first token (the Philox stream offset)."""
    return int(rank) * int(tokens_per_rank)


def allreduce_grad_w(dW, async_op=False):
    """Sum the per-shard grad_W partials over all ranks (NCCL over NVLink on
    B200; gloo on CPU test runs).  Returns the work handle if async_op."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return None
    return dist.all_reduce(dW, op=dist.ReduceOp.SUM, async_op=async_op)


def max_over_ranks(value, device):
    """Max of a scalar over ranks (step time: the job is as slow as its slowest rank)."""
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class SymmetricGradW:
    """A grad_W buffer in PyTorch symmetric memory with an NVLS multicast address
    (SURVEY.md §8(f4)): pass `multicast(offset)` as `dw_multicast` to
    Int4Linear.backward and the grad_W GEMM epilogue reduces its tiles into every
    rank's copy (multimem.red.add) -- no separate all-reduce pass.  Per step:
    zero_() on every rank before the backwards, barrier() after them.
    Plumbing only (allocation, rendezvous, barrier); the reduction runs in the
    library's kernel.  `available` is False when the device / driver offers no
    multicast object for this group (then use allreduce_grad_w)."""

    def __init__(self, numel, device, group=None):
        import torch.distributed._symmetric_memory as symm_mem
        group = group or dist.group.WORLD
        self.group_name = group.group_name
        try:
            symm_mem.enable_symm_mem_for_group(self.group_name)
        except Exception:
            pass
        self.tensor = symm_mem.empty(int(numel), dtype=torch.float32, device=device)
        self.handle = symm_mem.rendezvous(self.tensor, self.group_name)
        self.mc = int(getattr(self.handle, "multicast_ptr", 0) or 0)
        self.available = self.mc != 0

    def multicast(self, offset_elems=0):
        return self.mc + 4 * int(offset_elems)

    def zero_(self):
        self.tensor.zero_()

    def barrier(self):
        """Device-side barrier of the group on the current stream (every rank's
        reductions have landed in every copy once it returns on the device)."""
        self.handle.barrier(channel=0)
