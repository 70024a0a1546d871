"""FSD1 / FSV1 containers (io.py of the reference) on CPU, against files the reference wrote."""
import os

import numpy as np
import pytest

from conftest import ROOT

from paper_2311_16100_b200 import io as fio
from paper_2311_16100_b200.errors import DataError

GOLD = os.path.join(ROOT, "tests", "golden")


def test_read_reference_dataset_and_write_back_byte_identical(tmp_path):
    src = os.path.join(GOLD, "tiny_m8.fsd1")
    st = fio.read_dataset(src)
    assert st.spec.M == 8 and st.n_images == 5 and st.mask_radius == 3 and st.mode == "tri"
    assert st.images.shape == (5, 64) and st.images.dtype == np.complex128
    assert len(st.ctfs) == 5 and abs(st.ctfs[1].defocus - 1.3) < 1e-12
    out = fio.write_dataset(st, tmp_path / "copy.fsd1")
    assert open(out, "rb").read() == open(src, "rb").read()
    hdr = fio.read_dataset_header(src)
    assert hdr["N"] == 5 and hdr["interp_mode"] == "tri"


def test_read_reference_volume_and_write_back_byte_identical(tmp_path):
    src = os.path.join(GOLD, "tiny_m8.fsv1")
    vol = fio.read_volume(src)
    assert vol.spec.M == 8 and vol.values.shape == (512,)
    out = fio.write_volume(vol, tmp_path / "copy.fsv1")
    assert open(out, "rb").read() == open(src, "rb").read()


def test_corrupt_files_raise_data_error(tmp_path):
    raw = open(os.path.join(GOLD, "tiny_m8.fsd1"), "rb").read()
    bad = tmp_path / "bad.fsd1"
    bad.write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(DataError):
        fio.read_dataset(bad)
    bad.write_bytes(raw[:-16])  # truncated payload
    with pytest.raises(DataError):
        fio.read_dataset(bad)
    bad.write_bytes(raw[:10])  # truncated header
    with pytest.raises(DataError):
        fio.read_dataset(bad)
    with pytest.raises(DataError):
        fio.read_volume(tmp_path / "missing.fsv1")
