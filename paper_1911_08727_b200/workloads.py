"""Synthetic workloads of BASELINE.json's configs (gradient producers for the hot path).

Random-init models of the named architectures and synthetic batches of the named shapes (there
is no network for datasets or checkpoints).  The models are plain torch modules: they only
produce the gradients that LagsSGD sparsifies and exchanges.
"""

from __future__ import annotations

import torch


def resnet50(num_classes: int = 1000) -> torch.nn.Module:
    """Config 4: ResNet-50 (torchvision layout, 161 parameter tensors, 25,557,032 weights)."""
    import torchvision

    return torchvision.models.resnet50(num_classes=num_classes)


def resnet20(num_classes: int = 10) -> torch.nn.Module:
    """Config 2: CIFAR ResNet-20 (3 stages x 3 basic blocks, 16/32/64 channels)."""
    import torch.nn as nn

    class Block(nn.Module):
        def __init__(self, cin, cout, stride):
            super().__init__()
            self.c1 = nn.Conv2d(cin, cout, 3, stride, 1, bias=False)
            self.b1 = nn.BatchNorm2d(cout)
            self.c2 = nn.Conv2d(cout, cout, 3, 1, 1, bias=False)
            self.b2 = nn.BatchNorm2d(cout)
            self.short = None
            if stride != 1 or cin != cout:
                self.short = nn.Sequential(nn.Conv2d(cin, cout, 1, stride, bias=False), nn.BatchNorm2d(cout))

        def forward(self, x):
            y = torch.relu(self.b1(self.c1(x)))
            y = self.b2(self.c2(y))
            return torch.relu(y + (x if self.short is None else self.short(x)))

    layers = [nn.Conv2d(3, 16, 3, 1, 1, bias=False), nn.BatchNorm2d(16), nn.ReLU()]
    cin = 16
    for cout, stride in ((16, 1), (32, 2), (64, 2)):
        for i in range(3):
            layers.append(Block(cin, cout, stride if i == 0 else 1))
            cin = cout
    layers += [nn.AdaptiveAvgPool2d(1), nn.Flatten(), nn.Linear(64, num_classes)]
    return nn.Sequential(*layers)


def vgg16_cifar(num_classes: int = 10) -> torch.nn.Module:
    """Config 3: VGG-16 with batch norm for 32x32 inputs."""
    import torch.nn as nn

    cfg = [64, 64, "M", 128, 128, "M", 256, 256, 256, "M", 512, 512, 512, "M", 512, 512, 512, "M"]
    layers, cin = [], 3
    for c in cfg:
        if c == "M":
            layers.append(nn.MaxPool2d(2))
        else:
            layers += [nn.Conv2d(cin, c, 3, padding=1), nn.BatchNorm2d(c), nn.ReLU()]
            cin = c
    layers += [nn.Flatten(), nn.Linear(512, num_classes)]
    return nn.Sequential(*layers)


class LSTMPTB(torch.nn.Module):
    """Config 5: 2-layer LSTM language model, hidden 1500, vocab 10k (PTB-shaped, untied)."""

    def __init__(self, vocab: int = 10000, hidden: int = 1500, layers: int = 2):
        super().__init__()
        self.embed = torch.nn.Embedding(vocab, hidden)
        self.lstm = torch.nn.LSTM(hidden, hidden, layers)
        self.decoder = torch.nn.Linear(hidden, vocab)

    def forward(self, tokens):
        out, _ = self.lstm(self.embed(tokens))
        return self.decoder(out)


def synthetic_images(batch: int, size: int, classes: int, device, seed: int = 0):
    g = torch.Generator(device=device).manual_seed(seed)
    x = torch.randn(batch, 3, size, size, device=device, generator=g)
    y = torch.randint(0, classes, (batch,), device=device, generator=g)
    return x, y
