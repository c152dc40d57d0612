// forwards to the single B200 header (see wfc/wfc_b200.hpp): utf8_decode, utf8_valid, utf8_sanitize, utf8_append, is_unicode_space, is_word_char, simple_lower
#pragma once
#include "wfc/wfc_b200.hpp"
