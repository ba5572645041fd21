"""Copies the reference's six shipped run configurations (proj/configs/*.json)
into tests/golden/configs/ as test fixtures: the GPU box has no /root/reference,
and the drop-in test (tests/test_dropin_reference.py) runs each of them through
the reference's voxl::run and voxl::b200::run. Data only, byte for byte."""
import os
import shutil

SRC = "/root/reference/proj/configs"
DST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs")

if __name__ == "__main__":
    os.makedirs(DST, exist_ok=True)
    for name in sorted(os.listdir(SRC)):
        if name.endswith(".json"):
            shutil.copyfile(os.path.join(SRC, name), os.path.join(DST, name))
            print(name)
