"""Write paper_2103_15195_b200/data/gradsets.json: trainable-tensor sizes of the
torchvision Mask R-CNN R50-FPN and VGG-16 models in BACKPROP order (reversed
registration order), the shapes of BASELINE.json configs 4 and 5.  Needs
torchvision (present in this image); run once, the JSON is committed."""

import json
from pathlib import Path

import torchvision

OUT = Path(__file__).resolve().parents[1] / "paper_2103_15195_b200" / "data" / "gradsets.json"


def sizes(model):
    return [int(p.numel()) for p in model.parameters() if p.requires_grad][::-1]


def main():
    doc = {
        "maskrcnn_201": sizes(torchvision.models.detection.maskrcnn_resnet50_fpn(weights=None, weights_backbone=None)),
        "vgg16_32": sizes(torchvision.models.vgg16(weights=None)),
    }
    for k, v in doc.items():
        print(k, len(v), sum(v))
    OUT.write_text(json.dumps(doc))


if __name__ == "__main__":
    main()
