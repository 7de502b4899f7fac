"""Master-worker coordination baseline (§4.1,
Fig. 3a at PAPER.md:130): the strategy Bitvector Allreduce replaces, run for real across
processes so its per-cycle cost can be set beside `gr_step` (tools/bench_cfg4.py).

Every cycle ("tic"):
  (i)   each rank serializes its NEW requests (tensors that became pending since its last
        cycle; a request carries name/shape/dtype/op metadata) and rank 0 gathers
        them — MPI_Gatherv's two stages: a gather of the sizes, then the variable-size payloads;
  (ii)  rank 0 counts submissions per tensor (common = submitted by all N ranks);
  (iii) forms responses for common requests whose group is complete (Grouping),
        in first-submission order (R20/R21);
  (iv)  broadcasts the ordered response list — MPI_Bcast of the size, then of the payload.
The host CPU does all of it over a torch.distributed process group (gloo on CPU tensors, the
analogue of the paper's CPU-side MPI). Baseline code: not part of the product path, and it
shares no code with the oracle (oracle/master_worker.py) that the tests check it against.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

REQ_WORDS = 8   # one serialized request: 32 B (id, op, dtype, ndim, numel lo/hi, name hash lo/hi)
RESP_WORDS = 4  # one serialized response: 16 B (id, group, submitting-rank count, fused offset)


class MasterWorker:
    def __init__(self, rank: int, world_size: int, group_of, numel=None, pg=None):
        self.rank, self.N, self.pg = rank, world_size, pg
        self.group_of = np.asarray(group_of, dtype=np.int64)
        self.T = int(self.group_of.size)
        self.G = int(self.group_of.max()) + 1 if self.T else 0
        self.group_size = np.bincount(self.group_of, minlength=self.G)
        self.numel = np.asarray(numel if numel is not None else np.ones(self.T), dtype=np.int64)
        self._submitted = np.zeros(self.T, dtype=bool)  # this rank's requests this step
        self._executed = 0
        if rank == 0:
            self._count = np.zeros(self.T, dtype=np.int64)           # ranks that submitted t
            self._first = np.full(self.T, np.iinfo(np.int64).max)    # first-submission sequence
            self._seq = 0
            self._live = np.zeros(self.T, dtype=bool)                # submitted, not executed

    def _serialize(self, ids):
        rec = np.zeros((len(ids), REQ_WORDS), dtype=np.int32)
        if len(ids):
            t = np.asarray(ids, dtype=np.int64)
            rec[:, 0] = t
            rec[:, 1] = 0            # op: allreduce
            rec[:, 2] = 1            # dtype code
            rec[:, 3] = 1            # ndim
            rec[:, 4] = (self.numel[t] & 0x7FFFFFFF).astype(np.int32)
            rec[:, 5] = (self.numel[t] >> 31).astype(np.int32)
            rec[:, 6] = (t * 2654435761 & 0x7FFFFFFF).astype(np.int32)
        return torch.from_numpy(rec.reshape(-1))

    def cycle(self, new_ids):
        """One coordination cycle; every rank calls it with the tensors it marked since its
        previous call. Returns the ordered list of tensors to execute (identical on all ranks)
        and whether the step is complete (every tensor executed)."""
        new_ids = [int(t) for t in new_ids]
        for t in new_ids:
            if self._submitted[t]:
                raise RuntimeError(f"rank {self.rank}: tensor {t} submitted twice in one step")
            self._submitted[t] = True
        payload = self._serialize(new_ids)
        # (i) Gatherv: sizes, then payloads
        size = torch.tensor([len(new_ids)], dtype=torch.int64)
        if self.rank == 0:
            sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(self.N)]
            dist.gather(size, sizes, dst=0, group=self.pg)
            lists = [payload]
            for r in range(1, self.N):
                n = int(sizes[r])
                buf = torch.empty(n * REQ_WORDS, dtype=torch.int32)
                if n:
                    dist.recv(buf, src=r, group=self.pg)
                lists.append(buf)
            resp = self._coordinate(lists)
            head = torch.tensor([resp.shape[0]], dtype=torch.int64)
        else:
            dist.gather(size, None, dst=0, group=self.pg)
            if len(new_ids):
                dist.send(payload, dst=0, group=self.pg)
            head = torch.zeros(1, dtype=torch.int64)
        # (iv) Bcast: size, then the ordered responses
        dist.broadcast(head, src=0, group=self.pg)
        n = int(head)
        body = torch.from_numpy(resp.reshape(-1)) if self.rank == 0 else torch.empty(n * RESP_WORDS, dtype=torch.int32)
        if n:
            dist.broadcast(body, src=0, group=self.pg)
        ids = body.view(-1, RESP_WORDS)[:, 0].tolist() if n else []
        self._executed += n
        complete = self._executed == self.T
        if complete:
            self._reset()
        return ids, complete

    def _coordinate(self, lists):
        """(ii)-(iii) on rank 0."""
        for r, buf in enumerate(lists):
            ids = buf.view(-1, REQ_WORDS)[:, 0].numpy().astype(np.int64)
            new = ids[self._count[ids] == 0]  # first submissions, in this list's order
            self._first[new] = self._seq + np.arange(new.size)
            self._seq += new.size
            self._live[new] = True
            self._count[ids] += 1             # a rank never lists a tensor twice (checked at submit)
        common = self._live & (self._count == self.N)
        complete_groups = np.bincount(self.group_of[common], minlength=self.G) == self.group_size
        ready = np.flatnonzero(common & complete_groups[self.group_of])
        ready = ready[np.argsort(self._first[ready], kind="stable")]
        self._live[ready] = False
        resp = np.zeros((ready.size, RESP_WORDS), dtype=np.int32)
        resp[:, 0] = ready
        resp[:, 1] = self.group_of[ready]
        resp[:, 2] = self.N
        resp[:, 3] = np.cumsum(self.numel[ready]) - self.numel[ready] if ready.size else 0
        return resp

    def _reset(self):
        self._submitted[:] = False
        self._executed = 0
        if self.rank == 0:
            self._count[:] = 0
            self._first[:] = np.iinfo(np.int64).max
            self._seq = 0
            self._live[:] = False
