"""Activation capture for the prover (protocol.infer_and_capture).

Forward hooks keep every hooked module's output tensor on the device, on the stream the
forward ran on, so `prover_commit` can quantise and commit them without a host round trip
(the step before the prover path).
"""
from __future__ import annotations


class ActivationCapture:
    """Context manager: `with ActivationCapture(modules) as cap: out = model(x)`; then
    `cap.tensors` holds one activation tensor per hooked module call, in call order."""

    def __init__(self, modules):
        self.modules = list(modules)
        self.tensors = []
        self._handles = []

    def _hook(self, module, inputs, output):
        t = output[0] if isinstance(output, (tuple, list)) else output
        self.tensors.append(t.detach())

    def __enter__(self):
        self.tensors = []
        self._handles = [m.register_forward_hook(self._hook) for m in self.modules]
        return self

    def __exit__(self, *exc):
        for h in self._handles:
            h.remove()
        self._handles = []
        return False


def infer_and_capture(model, inputs, modules=None):
    """Run `model(inputs)` and return (output, activation tensors of `modules`).
    Default modules: the model's direct children (one tensor per layer)."""
    import torch

    mods = list(modules) if modules is not None else list(model.children())
    with ActivationCapture(mods) as cap, torch.no_grad():
        out = model(inputs)
    return out, cap.tensors
