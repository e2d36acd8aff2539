"""The BASELINE.json workloads (SURVEY.md §8 geometry table, §8d inputs).

Each entry: name -> (kernel r, stride s, pad, H=W, C_in, C_out, batch).
All use the reference's symmetric "same" padding r//2 except cfg3 (AlexNet
conv1, 227x227, pad 0 -> 55x55).
"""

from dataclasses import dataclass

from .convspec import ConvSpec


@dataclass(frozen=True)
class Workload:
    name: str
    kernel: int
    stride: int
    pad: int
    hw: int
    c_in: int
    c_out: int
    batch: int
    note: str = ""

    def spec(self) -> ConvSpec:
        return ConvSpec(kernel=(self.kernel, self.kernel), stride=(self.stride, self.stride),
                        pad=(self.pad,) * 4)

    def out_hw(self) -> tuple:
        return self.spec().out_dims(self.hw, self.hw)

    def direct_flops_per_image(self) -> int:
        """Direct-conv-equivalent FLOPs: 2 * C_in * C_out * OH * OW * r^2."""
        oh, ow = self.out_hw()
        return 2 * self.c_in * self.c_out * oh * ow * self.kernel * self.kernel


WORKLOADS = {
    w.name: w for w in [
        Workload("cfg1-5x5s1", 5, 1, 2, 56, 32, 32, 1, "single DWM conv2d, BASELINE configs[0]"),
        Workload("cfg2-resnet50-stem", 7, 2, 3, 224, 3, 64, 256, "ResNet-50 stem, BASELINE configs[1]"),
        Workload("cfg3-alexnet-conv1", 11, 4, 0, 227, 3, 96, 256, "AlexNet conv1, BASELINE configs[2]"),
        *[Workload(f"cfg4-{r}x{r}s1", r, 1, r // 2, 28, 256, 256, 512, "kernel sweep, BASELINE configs[3]")
          for r in (3, 5, 7, 9, 11)],
        *[Workload(f"cfg5-{r}x{r}s2", r, 2, r // 2, 56, 128, 256, 1024, "stride-2 sweep, BASELINE configs[4]")
          for r in (3, 5)],
    ]
}

DEFAULT_WORKLOAD = "cfg4-11x11s1"
