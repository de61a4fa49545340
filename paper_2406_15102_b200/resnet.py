"""ResNet-18 for CIFAR-10 (BASELINE configs[2]): torchvision's resnet18 with the
usual CIFAR stem (3x3 stride-1 conv, no max-pool) and a 10-way head.
``convert_resnet`` makes every Conv2d (HLQConv2d) and the Linear head
(HLQLinear) run the HLQ backward; the stem's input gradient is never needed,
so its dX is skipped."""
from __future__ import annotations

import torch.nn as nn

from .conv import convert_convs
from .layers import convert_linears


def resnet18_cifar(classes: int = 10) -> nn.Module:
    from torchvision.models import resnet18
    m = resnet18(num_classes=classes)
    m.conv1 = nn.Conv2d(3, 64, 3, stride=1, padding=1, bias=False)
    m.maxpool = nn.Identity()
    return m


def convert_resnet(model: nn.Module) -> nn.Module:
    return convert_linears(convert_convs(model))
