"""On-the-fly use of DF11 weights (NEXT-1): decompress a transformer block right before its
forward pass into a reused BF16 scratch, and prefetch the next block's decode on a side stream so that
it overlaps the current block's GEMMs.

    blocks = [BlockWeights.from_host([...HostTensor...], device) for each transformer block]
    runner = OverlapRunner(blocks, device)
    for i, weights in runner.iterate():       # weights: list of BF16 tensors (views into the scratch)
        x = forward_block(x, weights)         # runs on the current stream

The decode is the C-ABI `df11_decompress_block` (one launch per block); PyTorch provides the streams,
events and the scratch memory only.
"""
from __future__ import annotations

from . import df11


class BlockWeights:
    """The DF11 tensors of one transformer block, resident in HBM."""

    def __init__(self, dts):
        self.dts = list(dts)
        self.numel = sum(d.num_elements for d in self.dts)

    @classmethod
    def from_host(cls, hosts, device="cuda"):
        return cls([df11.to_device(h, device) for h in hosts])

    def plan(self, scratch):
        outs, o = [], 0
        for d in self.dts:
            outs.append(scratch[o:o + d.num_elements])
            o += (d.num_elements + 7) // 8 * 8
        return df11.BlockPlan(self.dts, outs)


class OverlapRunner:
    """Double-buffered BF16 scratch; block i+1 decodes on `decode_stream` while block i computes."""

    def __init__(self, blocks, device="cuda", prefetch: bool = True, decode_ctas: int = 0):
        """decode_ctas: SM budget of the prefetched decode (0 = every SM): the decode of block i+1
        then runs on that many SMs and leaves the rest to block i's GEMMs."""
        import torch
        self.blocks = list(blocks)
        self.device = torch.device(device)
        cap = max(b.numel + 8 * len(b.dts) for b in self.blocks) + 64
        self.scratch = [torch.empty(cap, dtype=torch.bfloat16, device=self.device) for _ in range(2)]
        self.prefetch = prefetch
        self.decode_ctas = int(decode_ctas)
        self.decode_stream = torch.cuda.Stream(device=self.device)
        self.plans = [[b.plan(self.scratch[k]) for k in range(2)] for b in self.blocks]
        self.decoded = [torch.cuda.Event() for _ in range(2)]
        self.consumed = [torch.cuda.Event() for _ in range(2)]

    def _decode(self, i, stream):
        import torch
        k = i % 2
        with torch.cuda.stream(stream):
            stream.wait_event(self.consumed[k])       # the scratch's previous block has been used
            self.plans[i][k].run(stream, max_ctas=self.decode_ctas if stream is self.decode_stream else 0)
            self.decoded[k].record(stream)

    def iterate(self):
        """Yield (i, [BF16 weight views]) in order; the yielded tensors are valid until the next step."""
        import torch
        main = torch.cuda.current_stream(self.device)
        n = len(self.blocks)
        for k in range(2):
            self.consumed[k].record(main)
        if n == 0:
            return
        self._decode(0, self.decode_stream if self.prefetch else main)
        for i in range(n):
            k = i % 2
            if self.prefetch and i + 1 < n:
                self._decode(i + 1, self.decode_stream)
            main.wait_event(self.decoded[k])
            outs = self.plans[i][k].outputs()
            yield i, [o.view(d.shape) for o, d in zip(outs, self.blocks[i].dts)]
            self.consumed[k].record(main)            # compute on this scratch is enqueued
            if not self.prefetch and i + 1 < n:
                self._decode(i + 1, main)
