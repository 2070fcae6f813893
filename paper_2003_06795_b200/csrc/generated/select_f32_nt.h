#ifndef SELECT_F32_NT_H
#define SELECT_F32_NT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_f32_nt_config;

static inline select_f32_nt_config select_f32_nt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(1792)) {
        if (m < INT64_C(159)) {
            if (k < INT64_C(544)) {
                if (k < INT64_C(405)) {
                    if (k < INT64_C(227)) {
                        if (m < INT64_C(113)) {
                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(70)) {
                            select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_nt_config out = {8u, 2u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(70)) {
                        select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                        return out;
                    } else {
                        select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                        return out;
                    }
                }
            } else {
                if (n < INT64_C(1432)) {
                    select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(28)) {
                        if (m < INT64_C(12)) {
                            select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(10138)) {
                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(70)) {
                            select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                            return out;
                        } else {
                            select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(351)) {
                if (m < INT64_C(555)) {
                    if (n < INT64_C(203)) {
                        if (k < INT64_C(272)) {
                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(702)) {
                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(1537)) {
                                if (m < INT64_C(278)) {
                                    if (k < INT64_C(992)) {
                                        select_f32_nt_config out = {8u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nt_config out = {8u, 2u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(176)) {
                        if (k < INT64_C(544)) {
                            if (m < INT64_C(1109)) {
                                if (k < INT64_C(314)) {
                                    select_f32_nt_config out = {8u, 2u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(444)) {
                                        select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {8u, 2u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(444)) {
                                    if (k < INT64_C(222)) {
                                        if (k < INT64_C(167)) {
                                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {8u, 2u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(314)) {
                                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(79)) {
                                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_f32_nt_config out = {8u, 2u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (k < INT64_C(702)) {
                                if (k < INT64_C(129)) {
                                    select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nt_config out = {8u, 2u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                            return out;
                        }
                    }
                }
            } else {
                if (m < INT64_C(1109)) {
                    if (n < INT64_C(1145)) {
                        if (m < INT64_C(634)) {
                            if (n < INT64_C(544)) {
                                if (m < INT64_C(448)) {
                                    if (k < INT64_C(3072)) {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {8u, 2u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(278)) {
                                    if (k < INT64_C(124)) {
                                        select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(203)) {
                                            select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(725)) {
                                if (k < INT64_C(144)) {
                                    select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(278)) {
                            if (k < INT64_C(405)) {
                                select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(725)) {
                                select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(768)) {
                        select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                        return out;
                    } else {
                        select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (m < INT64_C(35480)) {
            if (n < INT64_C(167)) {
                if (n < INT64_C(46)) {
                    if (m < INT64_C(17740)) {
                        if (k < INT64_C(118)) {
                            if (m < INT64_C(8870)) {
                                if (m < INT64_C(4435)) {
                                    select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(4435)) {
                                if (k < INT64_C(167)) {
                                    if (n < INT64_C(28)) {
                                        select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(8870)) {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(167)) {
                                        if (n < INT64_C(28)) {
                                            select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(8870)) {
                        if (k < INT64_C(40)) {
                            if (m < INT64_C(4435)) {
                                select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(544)) {
                                if (m < INT64_C(4435)) {
                                    if (n < INT64_C(111)) {
                                        if (k < INT64_C(111)) {
                                            select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(91)) {
                                        if (k < INT64_C(128)) {
                                            select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                            return out;
                                        }
                                    } else {
                                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (n < INT64_C(79)) {
                                    select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(79)) {
                            if (m < INT64_C(17740)) {
                                if (k < INT64_C(194)) {
                                    if (k < INT64_C(97)) {
                                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {8u, 4u, 4u, 8u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(194)) {
                                    select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(815)) {
                                select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(17740)) {
                                    select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(768)) {
                    if (m < INT64_C(4435)) {
                        if (n < INT64_C(363)) {
                            if (k < INT64_C(129)) {
                                select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                return out;
                            } else {
                                select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(111)) {
                                select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(91)) {
                            if (m < INT64_C(8870)) {
                                select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                return out;
                            }
                        } else {
                            if (k < INT64_C(182)) {
                                select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(17740)) {
                                    if (m < INT64_C(8870)) {
                                        if (n < INT64_C(363)) {
                                            select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (n < INT64_C(363)) {
                                            select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(2509)) {
                        select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                        return out;
                    } else {
                        select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                        return out;
                    }
                }
            }
        } else {
            if (n < INT64_C(46)) {
                select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                return out;
            } else {
                if (k < INT64_C(26)) {
                    select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                    return out;
                } else {
                    if (m < INT64_C(141920)) {
                        if (n < INT64_C(182)) {
                            if (k < INT64_C(97)) {
                                select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(384)) {
                                    select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(70960)) {
                                        select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(91)) {
                                            select_f32_nt_config out = {4u, 8u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                            return out;
                        }
                    } else {
                        select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                        return out;
                    }
                }
            }
        }
    }
}

#endif /* SELECT_F32_NT_H */
