"""TEST HELPER: lets the multi-rank DEVICE path (NCCL in production) run between processes that
share ONE GPU, over the gloo backend, by staging CUDA tensors through host memory inside
``torch.distributed``'s point-to-point and collective calls.  Product code is untouched -- the
shim patches the ``torch.distributed`` functions it calls.  None of the product's kernels waits
on another rank (all exchanges are host-driven collectives), so two time-sliced processes on one
GPU cannot deadlock on the device."""

import torch
import torch.distributed as dist


class _Work:
    def __init__(self, work, after=None):
        self.work, self.after = work, after

    def wait(self):
        self.work.wait()
        if self.after is not None:
            self.after()
            self.after = None
        return True


def install():
    o_send, o_recv, o_isend, o_irecv = dist.send, dist.recv, dist.isend, dist.irecv
    o_bcast, o_allgather, o_allreduce = dist.broadcast, dist.all_gather, dist.all_reduce

    def send(t, dst, group=None, tag=0):
        torch.cuda.synchronize()
        return o_send(t.cpu() if t.is_cuda else t, dst, group=group, tag=tag)

    def recv(t, src=None, group=None, tag=0):
        if not t.is_cuda:
            return o_recv(t, src, group=group, tag=tag)
        h = torch.empty(t.shape, dtype=t.dtype)
        r = o_recv(h, src, group=group, tag=tag)
        t.copy_(h)
        return r

    def isend(t, dst, group=None, tag=0):
        torch.cuda.synchronize()
        h = t.cpu() if t.is_cuda else t
        return _Work(o_isend(h, dst, group=group, tag=tag))

    def irecv(t, src=None, group=None, tag=0):
        if not t.is_cuda:
            return _Work(o_irecv(t, src, group=group, tag=tag))
        h = torch.empty(t.shape, dtype=t.dtype)
        return _Work(o_irecv(h, src, group=group, tag=tag), after=lambda: t.copy_(h))

    def batch_isend_irecv(ops):
        works = []
        for op in ops:
            fn = isend if op.op in (o_isend, isend) else irecv
            works.append(fn(op.tensor, op.peer, group=op.group, tag=op.tag))
        return works

    def broadcast(t, src, group=None, async_op=False):
        if not t.is_cuda:
            return o_bcast(t, src, group=group)
        torch.cuda.synchronize()
        h = t.cpu()
        o_bcast(h, src, group=group)
        t.copy_(h)

    def all_gather(out, t, group=None, async_op=False):
        if not t.is_cuda:
            return o_allgather(out, t, group=group)
        torch.cuda.synchronize()
        hs = [torch.empty(t.shape, dtype=t.dtype) for _ in out]
        o_allgather(hs, t.cpu(), group=group)
        for o, h in zip(out, hs):
            o.copy_(h)

    def all_reduce(t, op=dist.ReduceOp.SUM, group=None, async_op=False):
        if not t.is_cuda:
            return o_allreduce(t, op=op, group=group)
        torch.cuda.synchronize()
        h = t.cpu()
        o_allreduce(h, op=op, group=group)
        t.copy_(h)

    class P2POp:  # the real P2POp validates the op against the original functions
        def __init__(self, op, tensor, peer=None, group=None, tag=0, group_peer=None):
            self.op, self.tensor, self.peer, self.group, self.tag = op, tensor, peer, group, tag

    dist.send, dist.recv, dist.isend, dist.irecv = send, recv, isend, irecv
    dist.batch_isend_irecv, dist.P2POp = batch_isend_irecv, P2POp
    dist.broadcast, dist.all_gather, dist.all_reduce = broadcast, all_gather, all_reduce
