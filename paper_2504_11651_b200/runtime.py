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

    @property
    def vf(self) -> str:
        return self.dts[0].vf if self.dts else "bf16"

    def scratch_elements(self) -> int:
        """Words of a scratch that holds every tensor at a 16-byte aligned offset."""
        return self.numel + 16 * len(self.dts) + 64

    def plan(self, scratch):
        upv = 16 // scratch.element_size()                  # words per 16 bytes
        outs, o = [], 0
        for d in self.dts:
            outs.append(scratch[o:o + d.num_elements])
            o += (d.num_elements + upv - 1) // upv * upv    # 16-byte aligned views (128-bit stores)
        return df11.BlockPlan(self.dts, outs)


class OverlapRunner:
    """Double-buffered BF16 scratch; block i+1 decodes on `decode_stream` while block i computes."""

    def __init__(self, blocks, device="cuda", prefetch: bool = True, decode_ctas: int = 0):
        """decode_ctas: SM budget of the prefetched decode (0 = every SM): the decode of block i+1
        then runs on that many SMs and leaves the rest to block i's GEMMs."""
        import torch
        self.blocks = list(blocks)
        self.device = torch.device(device)
        cap = max(b.scratch_elements() for b in self.blocks) if self.blocks else 64
        dt = df11.out_dtype(self.blocks[0].vf if self.blocks else "bf16")
        self.scratch = [torch.empty(cap, dtype=dt, device=self.device) for _ in range(2)]
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


# --------------------------------------------------------------------------- PyTorch module hook
_VF_OF_DTYPE = {"torch.bfloat16": "bf16", "torch.float16": "fp16", "torch.float8_e4m3fn": "fp8_e4m3",
                "torch.float8_e5m2": "fp8_e5m2"}


class DF11Hook:
    """Thin PyTorch block hook (NEXT-1): the named weights of `module` live in HBM as DF11
    tensors only.  A forward pre-hook decodes them with ONE df11_decompress_block launch into a scratch
    and binds the views as the module's parameters; a forward hook unbinds them after the forward (the
    decoded matrices are "immediately discarded": the scratch can be shared by every block)."""

    def __init__(self, module, names, weights: BlockWeights, scratch=None):
        import torch
        self.module, self.names, self.weights = module, list(names), weights
        if scratch is None:
            dev = weights.dts[0].encoded_exponent.device
            scratch = torch.empty(weights.scratch_elements(), dtype=df11.out_dtype(weights.vf), device=dev)
        if scratch.numel() < weights.scratch_elements():
            raise ValueError("scratch too small for this block")
        self.plan = weights.plan(scratch)
        self.slots = []
        for n in self.names:
            path, _, attr = n.rpartition(".")
            sub = module.get_submodule(path) if path else module
            sub._parameters[attr] = None                 # the dense weight is dropped
            self.slots.append((sub, attr))
        self.handles = [module.register_forward_pre_hook(self._bind), module.register_forward_hook(self._unbind)]

    def _bind(self, mod, args):
        import torch
        self.plan.run()                                   # current stream, one launch
        for (sub, attr), w in zip(self.slots, self.plan.outputs()):
            sub._parameters[attr] = torch.nn.Parameter(w, requires_grad=False)

    def _unbind(self, mod, args, out):
        for sub, attr in self.slots:
            sub._parameters[attr] = None

    def remove(self):
        for h in self.handles:
            h.remove()


def encode_module(module, names=None, device="cuda", **encode_kw):
    """df11_encode the named parameters of `module` (default: every BF16 / FP16 / FP8 parameter) and
    upload them: returns (names, BlockWeights)."""
    if names is None:
        names = [n for n, p in module.named_parameters() if str(p.dtype) in _VF_OF_DTYPE]
    dts = []
    for n in names:
        p = module.get_parameter(n)
        h = df11.encode(p.detach().cpu(), vf=_VF_OF_DTYPE[str(p.dtype)], **encode_kw)
        dts.append(df11.to_device(h, device))
    return list(names), BlockWeights(dts)


def compress_module(module, names=None, device="cuda", scratch=None, **encode_kw) -> DF11Hook:
    """Encode the named parameters of `module` (default: every floating-point parameter of BF16 /
    FP16 / FP8 dtype) with df11_encode, keep only their DF11 form in HBM, and attach a DF11Hook."""
    names, weights = encode_module(module, names, device, **encode_kw)
    return DF11Hook(module, names, weights, scratch)


def compress_blocks(modules, device="cuda", **encode_kw):
    """The paper's deployment: the weights of every transformer block (and, passed as
    modules too, the embedding and the LM head) live in HBM as DF11 only; each module's forward is
    preceded by ONE batched decode of its weights into a scratch shared by all of them (the BF16
    matrices are "immediately discarded" after the forward).  Returns the hooks."""
    import torch
    encoded = [encode_module(m, None, device, **encode_kw) for m in modules]
    formats = {w.vf for _, w in encoded if w.dts}
    if len(formats) > 1:
        raise ValueError("one value format per model (the shared scratch has one dtype)")
    cap = max((w.scratch_elements() for _, w in encoded), default=64)
    scratch = torch.empty(cap, dtype=df11.out_dtype(formats.pop() if formats else "bf16"), device=device)
    return [DF11Hook(m, names, w, scratch) for m, (names, w) in zip(modules, encoded)]
