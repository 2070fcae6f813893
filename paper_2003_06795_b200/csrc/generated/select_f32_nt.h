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
            if (k < INT64_C(1145)) {
                if (n < INT64_C(1620)) {
                    if (k < INT64_C(430)) {
                        if (m < INT64_C(56)) {
                            select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(113)) {
                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(992)) {
                            if (m < INT64_C(70)) {
                                select_f32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(744)) {
                                    select_f32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (n < INT64_C(227)) {
                                        select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
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
                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                        return out;
                    }
                }
            } else {
                if (m < INT64_C(12)) {
                    select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                    return out;
                } else {
                    if (n < INT64_C(2024)) {
                        select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                        return out;
                    }
                }
            }
        } else {
            if (n < INT64_C(1145)) {
                if (n < INT64_C(287)) {
                    if (m < INT64_C(1109)) {
                        if (n < INT64_C(111)) {
                            if (m < INT64_C(278)) {
                                select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(272)) {
                                    if (k < INT64_C(167)) {
                                        select_f32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (n < INT64_C(79)) {
                                        select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(555)) {
                                            select_f32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        } else {
                            if (m < INT64_C(278)) {
                                if (n < INT64_C(203)) {
                                    if (k < INT64_C(744)) {
                                        select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(1537)) {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    } else {
                        if (k < INT64_C(314)) {
                            if (k < INT64_C(68)) {
                                select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            if (n < INT64_C(111)) {
                                select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                return out;
                            } else {
                                if (n < INT64_C(182)) {
                                    select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(278)) {
                        if (k < INT64_C(124)) {
                            if (k < INT64_C(79)) {
                                select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                return out;
                            }
                        } else {
                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (m < INT64_C(1109)) {
                            if (k < INT64_C(363)) {
                                if (m < INT64_C(555)) {
                                    select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    if (k < INT64_C(144)) {
                                        select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (m < INT64_C(448)) {
                                    if (k < INT64_C(992)) {
                                        select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (n < INT64_C(544)) {
                                if (k < INT64_C(91)) {
                                    select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (m < INT64_C(278)) {
                    if (k < INT64_C(405)) {
                        select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                        return out;
                    } else {
                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                        return out;
                    }
                } else {
                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                    return out;
                }
            }
        }
    } else {
        if (k < INT64_C(544)) {
            if (m < INT64_C(35480)) {
                if (n < INT64_C(167)) {
                    if (m < INT64_C(17740)) {
                        if (n < INT64_C(46)) {
                            if (m < INT64_C(8870)) {
                                if (m < INT64_C(4435)) {
                                    if (n < INT64_C(28)) {
                                        select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(167)) {
                                            select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                            return out;
                                        }
                                    }
                                } else {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(167)) {
                                    if (n < INT64_C(20)) {
                                        select_f32_nt_config out = {4u, 2u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                        return out;
                                    }
                                } else {
                                    select_f32_nt_config out = {2u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (n < INT64_C(111)) {
                                if (k < INT64_C(222)) {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(4435)) {
                                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(8870)) {
                                            select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(4435)) {
                                    select_f32_nt_config out = {4u, 4u, 2u, 8u, 16u};
                                    return out;
                                } else {
                                    if (m < INT64_C(8870)) {
                                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(363)) {
                                            select_f32_nt_config out = {2u, 8u, 4u, 16u, 8u};
                                            return out;
                                        } else {
                                            select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(46)) {
                            select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                            return out;
                        } else {
                            select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        }
                    }
                } else {
                    if (m < INT64_C(8870)) {
                        if (n < INT64_C(768)) {
                            if (m < INT64_C(4435)) {
                                if (k < INT64_C(111)) {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(363)) {
                                        select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(65)) {
                                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(182)) {
                                        select_f32_nt_config out = {2u, 8u, 4u, 16u, 8u};
                                        return out;
                                    } else {
                                        select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                            return out;
                        }
                    } else {
                        select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                        return out;
                    }
                }
            } else {
                if (k < INT64_C(146)) {
                    if (m < INT64_C(283839)) {
                        if (k < INT64_C(30)) {
                            if (m < INT64_C(141920)) {
                                select_f32_nt_config out = {2u, 8u, 4u, 16u, 8u};
                                return out;
                            } else {
                                select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                return out;
                            }
                        } else {
                            select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
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
        } else {
            if (m < INT64_C(17740)) {
                if (n < INT64_C(363)) {
                    if (m < INT64_C(4435)) {
                        select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (n < INT64_C(91)) {
                            select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(8870)) {
                                if (n < INT64_C(182)) {
                                    select_f32_nt_config out = {2u, 4u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            } else {
                                if (n < INT64_C(182)) {
                                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (n < INT64_C(2509)) {
                        if (m < INT64_C(4435)) {
                            select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(8870)) {
                                select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(3259)) {
                                    select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                                    return out;
                                } else {
                                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
                                }
                            }
                        }
                    } else {
                        select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                        return out;
                    }
                }
            } else {
                if (m < INT64_C(141920)) {
                    if (n < INT64_C(91)) {
                        select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(35480)) {
                            select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                            return out;
                        } else {
                            if (m < INT64_C(70960)) {
                                if (k < INT64_C(1630)) {
                                    select_f32_nt_config out = {8u, 8u, 4u, 16u, 8u};
                                    return out;
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
                } else {
                    select_f32_nt_config out = {8u, 8u, 8u, 16u, 8u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_F32_NT_H */
