#ifndef SELECT_BF16_NT_H
#define SELECT_BF16_NT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_bf16_nt_config;

static inline select_bf16_nt_config select_bf16_nt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (k < INT64_C(1087)) {
        if (m < INT64_C(35480)) {
            if (m < INT64_C(4435)) {
                if (n < INT64_C(992)) {
                    if (k < INT64_C(744)) {
                        if (m < INT64_C(2218)) {
                            if (m < INT64_C(113)) {
                                if (k < INT64_C(304)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(314)) {
                                    if (n < INT64_C(46)) {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(91)) {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(111)) {
                                                if (m < INT64_C(1109)) {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(46)) {
                                                        select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        if (k < INT64_C(79)) {
                                                            select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    }
                                                }
                                            } else {
                                                if (m < INT64_C(159)) {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (m < INT64_C(278)) {
                                                        select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    } else {
                                                        if (m < INT64_C(555)) {
                                                            select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            if (n < INT64_C(702)) {
                                                                if (m < INT64_C(1109)) {
                                                                    if (k < INT64_C(182)) {
                                                                        select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                                                        return out;
                                                                    } else {
                                                                        select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                                                        return out;
                                                                    }
                                                                } else {
                                                                    if (k < INT64_C(182)) {
                                                                        select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                                                        return out;
                                                                    } else {
                                                                        if (n < INT64_C(257)) {
                                                                            select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                                                            return out;
                                                                        } else {
                                                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                                            return out;
                                                                        }
                                                                    }
                                                                }
                                                            } else {
                                                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            }
                                                        }
                                                    }
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(448)) {
                                        if (k < INT64_C(444)) {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(544)) {
                                                if (m < INT64_C(278)) {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (n < INT64_C(124)) {
                                                    if (m < INT64_C(278)) {
                                                        select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        if (k < INT64_C(444)) {
                                            if (n < INT64_C(79)) {
                                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (n < INT64_C(544)) {
                                if (n < INT64_C(363)) {
                                    if (n < INT64_C(167)) {
                                        if (k < INT64_C(79)) {
                                            select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(314)) {
                                                if (k < INT64_C(222)) {
                                                    if (k < INT64_C(167)) {
                                                        if (k < INT64_C(118)) {
                                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            if (n < INT64_C(28)) {
                                                                select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                                                return out;
                                                            }
                                                        }
                                                    } else {
                                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(544)) {
                                                    select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (m < INT64_C(555)) {
                                if (m < INT64_C(278)) {
                                    if (n < INT64_C(287)) {
                                        if (m < INT64_C(70)) {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(992)) {
                                            select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(70)) {
                                                select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(139)) {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    if (n < INT64_C(287)) {
                                        select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(992)) {
                                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (n < INT64_C(203)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            select_bf16_nt_config out = {8u, 1u, 4u, 8u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(278)) {
                        if (k < INT64_C(405)) {
                            if (k < INT64_C(287)) {
                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(70)) {
                                select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(139)) {
                                    if (k < INT64_C(725)) {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(725)) {
                                        select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        }
                    } else {
                        if (k < INT64_C(405)) {
                            if (m < INT64_C(1109)) {
                                select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(555)) {
                                if (n < INT64_C(1449)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(111)) {
                    if (k < INT64_C(79)) {
                        if (m < INT64_C(8870)) {
                            select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                            return out;
                        } else {
                            if (n < INT64_C(23)) {
                                if (m < INT64_C(17740)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(222)) {
                            if (n < INT64_C(28)) {
                                if (m < INT64_C(8870)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        } else {
                            if (m < INT64_C(17740)) {
                                if (m < INT64_C(8870)) {
                                    if (k < INT64_C(384)) {
                                        select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(46)) {
                        if (m < INT64_C(8870)) {
                            select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(17740)) {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        if (m < INT64_C(8870)) {
                            if (n < INT64_C(257)) {
                                if (k < INT64_C(363)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    }
                }
            }
        } else {
            if (n < INT64_C(46)) {
                if (n < INT64_C(20)) {
                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    if (k < INT64_C(118)) {
                        if (m < INT64_C(70960)) {
                            select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(141920)) {
                                select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                        return out;
                    }
                }
            } else {
                if (n < INT64_C(111)) {
                    if (m < INT64_C(70960)) {
                        if (k < INT64_C(97)) {
                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(194)) {
                                select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(70960)) {
                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        }
    } else {
        if (n < INT64_C(1432)) {
            if (m < INT64_C(1109)) {
                if (m < INT64_C(28)) {
                    if (k < INT64_C(2897)) {
                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(6)) {
                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(12)) {
                                select_bf16_nt_config out = {8u, 1u, 4u, 8u, 8u};
                                return out;
                            } else {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(555)) {
                        if (n < INT64_C(363)) {
                            select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(139)) {
                                if (k < INT64_C(3072)) {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                if (m < INT64_C(278)) {
                                    if (k < INT64_C(3072)) {
                                        select_bf16_nt_config out = {4u, 1u, 1u, 16u, 16u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(363)) {
                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nt_config out = {8u, 1u, 4u, 8u, 8u};
                            return out;
                        }
                    }
                }
            } else {
                if (k < INT64_C(1630)) {
                    if (m < INT64_C(35480)) {
                        if (m < INT64_C(8870)) {
                            if (m < INT64_C(2218)) {
                                select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                if (m < INT64_C(4435)) {
                                    select_bf16_nt_config out = {8u, 1u, 4u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(182)) {
                                        select_bf16_nt_config out = {8u, 1u, 4u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_bf16_nt_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    if (m < INT64_C(2218)) {
                        if (n < INT64_C(363)) {
                            select_bf16_nt_config out = {8u, 1u, 4u, 8u, 8u};
                            return out;
                        } else {
                            select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(4435)) {
                            select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                            return out;
                        } else {
                            if (m < INT64_C(17740)) {
                                if (k < INT64_C(3259)) {
                                    select_bf16_nt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            } else {
                                select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                                return out;
                            }
                        }
                    }
                }
            }
        } else {
            if (m < INT64_C(6)) {
                if (k < INT64_C(10138)) {
                    select_bf16_nt_config out = {8u, 1u, 4u, 8u, 8u};
                    return out;
                } else {
                    select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                select_bf16_nt_config out = {4u, 1u, 8u, 16u, 16u};
                return out;
            }
        }
    }
}

#endif /* SELECT_BF16_NT_H */
