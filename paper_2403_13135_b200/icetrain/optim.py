"""Adam facade over the fused ice_adam kernel (torch.optim.Adam defaults, train.py:149)."""
from __future__ import annotations


class Adam:
    """Drop-in for ``torch.optim.Adam(model.parameters(), lr=...)`` on a B200 UNet, fused into
    one ice_adam pass over the flat buffers (+ the bf16 working copy, + gradient zeroing).
    ``params`` is what UNet.parameters() returns.  torch.optim.Adam on the same parameters
    also works (unfused: see train.synchronized_step)."""

    def __init__(self, params, lr: float = 1e-3, betas=(0.9, 0.999), eps: float = 1e-8,
                 weight_decay: float = 0.0, amsgrad: bool = False):
        if lr <= 0:
            raise ValueError(f"Invalid learning rate: {lr}")
        if weight_decay or amsgrad:
            raise ValueError("only the reference's Adam defaults (no weight decay, no amsgrad) are fused")
        engine = getattr(params, "engine", None)  # UNet.parameters() (a ParamList)
        if engine is not None:
            self.engines = [engine]
        else:
            self.engines = list(params)
            if not all(hasattr(e, "adam_slice") for e in self.engines):
                raise TypeError("icetrain.Adam steps a B200 UNet's parameters(): pass model.parameters() "
                                "(use torch.optim.* for arbitrary tensors)")
        self.lr, self.betas, self.eps = lr, tuple(betas), eps
        self.step_count = 0

    def step(self) -> None:
        self.step_count += 1
        for e in self.engines:
            e.adam(self.step_count, self.lr, self.betas, self.eps)

    # ---- optimizer-in-backward (used by train.StepOverlap): the step count advances once,
    # then each gradient bucket is updated as soon as it is final, on a side stream
    def begin_overlapped_step(self) -> int:
        self.step_count += 1
        for e in self.engines:
            e.advance_step()
        return self.step_count

    def step_slice(self, engine, start: int, stop: int, stream=None) -> None:
        engine.adam_slice(start, stop, self.step_count, self.lr, self.betas, self.eps, stream)

    def zero_grad(self, set_to_none: bool = True) -> None:
        for e in self.engines:
            e.zero_grad()
