"""The reference's catalog tables (pure Python: no native library, so the
bench's reference arm can name the same models without loading libtrims.so).
Restates proj/src/bench/catalog.cpp:21-66 (the paper's Table 2 / Table 4 rows).
"""

# name, layers, workspace MB, weights MB  (catalog.cpp:21-59)
SMALL37 = [
    ("alexnet", 16, 516, 238), ("googlenet", 116, 111, 27), ("caffenet", 16, 512, 233),
    ("rcnn-ilsvrc13", 16, 479, 221), ("dpn68", 361, 122, 49), ("dpn92", 481, 340, 145),
    ("inception-v3", 472, 257, 92), ("inception-v4", 747, 399, 164), ("inceptionbn-v2", 416, 313, 129),
    ("inceptionbn-v3", 416, 142, 44), ("inception-resnet-v2", 1102, 493, 214), ("locationnet", 514, 666, 285),
    ("nin", 24, 131, 29), ("resnet101", 526, 423, 170), ("resnet101-v2", 522, 428, 171),
    ("resnet152", 777, 548, 231), ("resnet152-11k", 769, 721, 311), ("resnet152-v2", 761, 340, 231),
    ("resnet18-v2", 99, 154, 45), ("resnet200-v2", 1009, 589, 248), ("resnet269-v2", 1346, 889, 391),
    ("resnet34-v2", 179, 222, 84), ("resnet50", 268, 270, 98), ("resnet50-v2", 259, 275, 98),
    ("resnext101", 526, 375, 170), ("resnext101-32x4d", 522, 378, 170), ("resnext26-32x4d", 147, 147, 59),
    ("resnext50", 271, 222, 96), ("resnext50-32x4d", 267, 224, 96), ("squeezenet-v1.0", 52, 34, 4.8),
    ("squeezenet-v1.1", 52, 28, 4.8), ("vgg16", 32, 1228, 528), ("vgg16-sod", 32, 1198, 514),
    ("vgg16-sos", 32, 1195, 513), ("vgg19", 38, 1270, 549), ("wrn50-v2", 267, 758, 264),
    ("xception", 236, 244, 88),
]
# catalog.cpp:62-66 (no workspace figures in the source table)
LARGE8 = [("alexnet-s1", 16, 0, 238), ("alexnet-s2", 16, 0, 770), ("alexnet-s3", 16, 0, 1694),
          ("alexnet-s4", 16, 0, 3010), ("vgg16-s1", 32, 0, 528), ("vgg16-s2", 32, 0, 1704),
          ("vgg16-s3", 32, 0, 3664), ("vgg16-s4", 32, 0, 6408)]
